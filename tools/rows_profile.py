"""Per-level timeline of the row-partitioned engine with G virtual ranks on one GPU (fused
p2p protocol, one launch): stage 1, exchange (2a + cross-rank barrier), whole-frontier
sweep (2b), per rank-0 timestamps; and the local queue of every rank.

    python tools/rows_profile.py --config c2 --ranks 8 [--sources 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--ranks", type=int, default=8)
    ap.add_argument("--sources", type=int, default=2)
    args = ap.parse_args()
    import numpy as np
    import torch
    import bench
    from paper_2512_21967_b200 import multigpu as MG
    torch.cuda.set_device(0)
    prep = bench.prepare(args.config, None, 1 << 16, build=False)
    gp, perm = prep["gp"], prep["perm"]
    bounds, slices = MG.partition_rows(gp, args.ranks)
    engs = [MG.RowsEngine(gp, r, args.ranks, bounds) for r in range(args.ranks)]
    MG.set_local_peers(engs)
    srcs = prep["g"].pick_sources(args.sources + 1, 1)
    if not perm.is_identity():
        srcs = perm.forward_map()[srcs]
    out = dict(config=args.config, ranks=args.ranks, vss=[e.num_vss for e in engs], slices=slices, runs=[])
    for s in srcs:
        for _ in range(2):
            MG.group_bfs(engs, int(s))
            res = [e.finish(False) for e in engs]
            torch.cuda.synchronize()
        t = engs[0].phase_times()
        lv = []
        for i, row in enumerate(t):
            a, b, c, d = [int(x) for x in row]
            lv.append(dict(level=i + 1, stage1_us=round((b - a) / 1e3, 1), exch_us=round((c - b) / 1e3, 1),
                           sweep_us=round((d - c) / 1e3, 1), level_us=round((d - a) / 1e3, 1)))
        total = (int(t[-1][3]) - int(t[0][0])) / 1e3 if len(t) else 0
        out["runs"].append(dict(source=int(s), total_us=round(total, 1), levels=lv,
                                queue_per_rank=[r.queue for r in res]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
