"""Per-level device timeline of the fused BFS kernel (from %globaltimer stamps the kernel
records at each grid barrier): queue size, discoveries, stage-1 / stage-2 / level time,
and the per-level algorithmic bytes over the level time.

    python tools/phase_profile.py --config c2 [--mode lazy] [--pull popc] [--sources 3]
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--pull", default="popc")
    ap.add_argument("--order", default=None)
    ap.add_argument("--sources", type=int, default=3)
    ap.add_argument("--grid-ctas", type=int, default=0)
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    import bench
    import paper_2512_21967_b200 as B
    from paper_2512_21967_b200 import _lib as L
    prep = bench.prepare(args.config, args.order, 1 << 16)
    b, g, plan, perm = prep["b"], prep["g"], prep["plan"], prep["perm"]
    mode = B.choose_mode(b, plan, B.EngineConfig(mode=B.engine_mode_from_string(args.mode)))
    lib = L.lib()
    ecfg = L.EngineConfigT(L.MODE_LAZY if mode == B.EngineMode.Lazy else L.MODE_EAGER,
                           L.PULL_MMA if args.pull == "mma" else L.PULL_POPC, 0, 0, args.grid_ctas, args.threads)
    srcs = g.pick_sources(args.sources, 1)
    if not perm.is_identity():
        srcs = perm.forward_map()[srcs]
    cap = 1 << 16
    tr = (L.LevelTraceT * cap)()
    ts = (C.c_uint64 * (3 * cap))()
    ctr = L.CountersT()
    out = []
    for s in srcs:
        for _ in range(2):  # second run is the one reported (warm)
            L.check(lib.blest_bfs(b.handle, int(s), C.byref(ecfg), None, C.byref(ctr),
                                  C.cast(tr, C.c_void_p), cap))
        rows = C.c_uint32()
        L.check(lib.blest_bfs_phase_times(b.handle, C.cast(ts, C.c_void_p), cap, C.byref(rows)))
        levels = []
        for i in range(min(rows.value, 64)):
            t0, t1, t2 = ts[3 * i], ts[3 * i + 1], ts[3 * i + 2]
            q = tr[i].queue_size
            s1 = (t1 - t0) / 1e3 if t1 else None
            tot = (t2 - t0) / 1e3
            levels.append(dict(level=i + 1, queue=q, discovered=tr[i].discovered, pushes=tr[i].queue_pushes,
                               relaxed=tr[i].relaxed_atomics, full=tr[i].full_atomics,
                               stage1_us=round(s1, 2) if s1 is not None else None,
                               level_us=round(tot, 2), vss_GBps=round(648 * q / (tot * 1e3), 1) if tot else None))
        total_us = (ts[3 * (rows.value - 1) + 2] - ts[0]) / 1e3 if rows.value else 0
        # every level, bucketed by queue size (high-diameter graphs: where the time goes)
        hist = {}
        for i in range(min(rows.value, cap)):
            q = tr[i].queue_size
            k = 0 if q == 0 else q.bit_length()
            h = hist.setdefault(k, [0, 0.0, 0.0, 0])
            h[0] += 1
            h[1] += (ts[3 * i + 2] - ts[3 * i]) / 1e3
            h[2] += ((ts[3 * i + 1] - ts[3 * i]) / 1e3) if ts[3 * i + 1] else 0.0
            h[3] += q
        buckets = [dict(queue_lt=1 << k, levels=h[0], total_us=round(h[1], 1), mean_level_us=round(h[1] / h[0], 2),
                        mean_stage1_us=round(h[2] / h[0], 2), mean_queue=round(h[3] / h[0], 1))
                   for k, h in sorted(hist.items())]
        out.append(dict(source=int(s), engine=mode.value, levels=levels, total_us=round(total_us, 2),
                        dequeues=ctr.vss_dequeues, iterations=rows.value, queue_buckets=buckets))
    print(json.dumps(dict(config=args.config, n=b.n, num_vss=b.num_vss, runs=out), indent=1))


if __name__ == "__main__":
    main()
