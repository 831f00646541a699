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
    ap.add_argument("--compare-lazy", action="store_true", help="also the single-GPU lazy engine (σ off/on)")
    args = ap.parse_args()
    import numpy as np
    import torch
    import bench
    from paper_2512_21967_b200 import multigpu as MG
    torch.cuda.set_device(0)
    prep = bench.prepare(args.config, None, 1 << 16, build=args.compare_lazy)
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
    if args.compare_lazy:
        import ctypes as C
        from paper_2512_21967_b200 import _lib as L
        lib = L.lib()
        b = prep["b"]
        ecfg = L.EngineConfigT(L.MODE_LAZY, L.PULL_POPC, 0, 0, 0, 0)
        ctr = L.CountersT()
        cap = 64
        ts = (C.c_uint64 * (3 * cap))()
        out["lazy"] = {}
        for sig in ("0", "1"):
            os.environ["BLEST_SIGMA"] = sig
            runs = []
            for s in srcs:
                for _ in range(2):
                    L.check(lib.blest_bfs(b.handle, int(s), C.byref(ecfg), None, C.byref(ctr), None, 0))
                rows = C.c_uint32()
                L.check(lib.blest_bfs_phase_times(b.handle, C.cast(ts, C.c_void_p), cap, C.byref(rows)))
                lv = [(i + 1, round((ts[3 * i + 1] - ts[3 * i]) / 1e3, 1) if ts[3 * i + 1] else None,
                       round((ts[3 * i + 2] - ts[3 * i]) / 1e3, 1)) for i in range(rows.value)]
                runs.append(dict(source=int(s), total_us=round((ts[3 * (rows.value - 1) + 2] - ts[0]) / 1e3, 1), levels=lv))
            out["lazy"]["sigma" + sig] = runs
        os.environ.pop("BLEST_SIGMA")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
