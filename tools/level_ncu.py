"""Isolate one BFS level for ncu: runs the same source with the level cap at L-1 and at L
(the capped run stops with the runaway status, which is caught), so the difference of the
two profiled launches is level L. Usage under ncu:
    ncu --set full -k regex:k_bfs -o out python tools/level_ncu.py --config c2 --level 4
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--mode", default="auto")
    ap.add_argument("--level", type=int, default=4)
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    import bench
    import paper_2512_21967_b200 as B
    from paper_2512_21967_b200 import _lib as L
    prep = bench.prepare(args.config, None, 1 << 16)
    b, g, plan, perm = prep["b"], prep["g"], prep["plan"], prep["perm"]
    mode = B.choose_mode(b, plan, B.EngineConfig(mode=B.engine_mode_from_string(args.mode)))
    lib = L.lib()
    src = g.pick_sources(1, 1)
    if not perm.is_identity():
        src = perm.forward_map()[src]
    ctr = L.CountersT()
    for cap in (args.level - 1, args.level):
        ecfg = L.EngineConfigT(L.MODE_LAZY if mode == B.EngineMode.Lazy else L.MODE_EAGER, L.PULL_POPC,
                               cap, 0, 0, args.threads)
        rc = lib.blest_bfs(b.handle, int(src[0]), C.byref(ecfg), None, C.byref(ctr), None, 0)
        print(f"cap {cap}: rc {rc}", file=sys.stderr)


if __name__ == "__main__":
    main()
