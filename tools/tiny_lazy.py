import sys, numpy as np
sys.path.insert(0, '.')
import paper_2512_21967_b200 as B
g = B.Graph.from_edges(300, np.stack([np.arange(299), np.arange(1, 300)], 1), directed=False)
b = B.build_bvss(g)
r, c = B.run_lazy(b, 0)
print("ok", r.levels[:10], c.vss_dequeues)
