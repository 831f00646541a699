"""Same-process A/B of engine switches (environment variables read at each launch) on one
prepared structure: every variant times the same sources, interleaved over rounds, so box
and clock drift hit all variants alike. Prints one JSON document: per variant the mean ms
per BFS, the harmonic-mean GTEPS and the per-level timeline of the first source.

    python tools/ab.py --config c2 --variants '{"masked": {}, "plain": {"BLEST_XFLAGS": "128"}}'
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
    ap.add_argument("--mode", default="b200")
    ap.add_argument("--sources", type=int, default=8)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--variants", required=True, help="JSON {name: {ENV: value}}")
    ap.add_argument("--levels", action="store_true", help="per-level timeline of the first source")
    args = ap.parse_args()
    import numpy as np
    import torch
    import bench
    import paper_2512_21967_b200 as B
    from paper_2512_21967_b200 import _lib as L
    torch.cuda.set_device(0)
    lib = L.lib()
    stream = torch.cuda.current_stream()
    L.check(lib.blest_set_stream(C.c_void_p(stream.cuda_stream)))
    variants = json.loads(args.variants)
    prep = bench.prepare(args.config, None, 1 << 16)
    b, g, plan, perm = prep["b"], prep["g"], prep["plan"], prep["perm"]
    if args.mode == "b200":
        lazy = bench.engine_policy_lazy(b.n, b.m, b.num_vss)
    else:
        lazy = B.choose_mode(b, plan, B.EngineConfig(mode=B.engine_mode_from_string(args.mode))) == B.EngineMode.Lazy
    ecfg = L.EngineConfigT(L.MODE_LAZY if lazy else L.MODE_EAGER, L.PULL_POPC, 0, 0, 0, 0)
    srcs = g.pick_sources(args.sources + 2, 1)
    if not perm.is_identity():
        srcs = perm.forward_map()[srcs]
    ctr = L.CountersT()
    ebytes = C.c_uint64()
    L.check(lib.blest_bfs_prepare(b.handle, C.byref(ecfg), C.byref(ebytes)))
    census = bench.census_of(lib, L, b, prep, srcs[2:], lazy, "popc", 0, 0, keep_levels=set())
    E = np.array([c["E"] for c in census], np.float64)
    base_env = dict(os.environ)
    times = {k: [] for k in variants}
    for _ in range(args.rounds):
        for name, env in variants.items():
            os.environ.clear()
            os.environ.update(base_env)
            os.environ.update({k: str(v) for k, v in env.items()})
            for s in srcs[:2]:  # warm-up under this variant
                L.check(lib.blest_bfs(b.handle, int(s), C.byref(ecfg), None, C.byref(ctr), None, 0))
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in srcs[2:]]
            torch.cuda.synchronize()
            for (e0, e1), s in zip(ev, srcs[2:]):
                e0.record(stream)
                L.check(lib.blest_bfs_launch(b.handle, int(s), C.byref(ecfg)))
                e1.record(stream)
            torch.cuda.synchronize()
            L.check(lib.blest_bfs_finish(b.handle, None, C.byref(ctr), None, 0))
            times[name].append([a.elapsed_time(z) / 1e3 for a, z in ev])
    out = dict(config=args.config, engine="lazy" if lazy else "eager", n=b.n, num_vss=b.num_vss, variants={})
    for name, env in variants.items():
        t = np.array(times[name])  # rounds x sources
        per_round_hm = [len(r) / float(np.sum(r / E)) / 1e9 for r in t]
        rec = dict(env=env, ms_mean=round(float(t.mean()) * 1e3, 4), ms_round_means=[round(float(r.mean()) * 1e3, 4) for r in t],
                   gteps_hm=round(float(np.mean(per_round_hm)), 2))
        if args.levels:
            os.environ.clear()
            os.environ.update(base_env)
            os.environ.update({k: str(v) for k, v in env.items()})
            cap = 1 << 12
            tr = (L.LevelTraceT * cap)()
            ts = (C.c_uint64 * (3 * cap))()
            for _ in range(2):
                L.check(lib.blest_bfs(b.handle, int(srcs[2]), C.byref(ecfg), None, C.byref(ctr), C.cast(tr, C.c_void_p), cap))
            rows = C.c_uint32()
            L.check(lib.blest_bfs_phase_times(b.handle, C.cast(ts, C.c_void_p), cap, C.byref(rows)))
            lv = []
            for i in range(min(rows.value, 16)):
                t0, t1, t2 = ts[3 * i], ts[3 * i + 1], ts[3 * i + 2]
                lv.append(dict(level=i + 1, queue=tr[i].queue_size, disc=tr[i].discovered,
                               s1_us=round((t1 - t0) / 1e3, 1) if t1 else None, us=round((t2 - t0) / 1e3, 1)))
            rec["levels"] = lv
        out["variants"][name] = rec
    os.environ.clear()
    os.environ.update(base_env)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
