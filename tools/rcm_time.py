import sys, time
sys.path.insert(0, '/root/repo')
import bench
import paper_2512_21967_b200 as B
kind, prm, ordering, desc = bench.CONFIGS[sys.argv[1]]
t=time.time()
if kind == "grid": g = B.Graph.generate_grid(prm["rows"], prm["cols"])
else:
    n = 1 << prm["scale"]; g = B.Graph.generate_urand(n, prm["ef"] * n, prm["seed"])
if prm.get("relabel") is not None:
    g = B.apply_permutation(g, B.relabel_permutation(g.num_vertices(), prm["relabel"]))
print("gen", time.time()-t, flush=True)
t=time.time(); r=B.classify_social_like(g); print("classify", time.time()-t, flush=True)
for _ in range(2):
    t=time.time(); p=B.rcm(g); print("rcm", time.time()-t, flush=True)
import numpy as np, ctypes as C
from paper_2512_21967_b200 import _lib as L
f = np.zeros(g.num_vertices(), np.uint32)
t=time.time(); L.check(L.lib().blest_order_rcm(g.handle, f.ctypes.data)); print("abi rcm", time.time()-t, flush=True)
t=time.time(); P=B.Permutation(f); print("Permutation()", time.time()-t, flush=True)
