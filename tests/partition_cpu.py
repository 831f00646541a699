"""TEST INFRASTRUCTURE: a numpy backend of the row-partitioned BFS protocol
(paper_2512_21967_b200/multigpu.py), built on the oracle's BVSS builder over the
row-filtered graph. Used by the gloo (CPU, world_size 2) tests of the multi-GPU host logic."""
import numpy as np
import torch

import oracle as O

INF = 0xFFFFFFFF


def rows_graph(g, lo, hi):
    """Arcs of g whose target lies in [lo, hi) (the rank's slice of A)."""
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.offsets).astype(np.int64))
    keep = (g.targets >= lo) & (g.targets < hi)
    return O.from_edges(g.n, src[keep], g.targets[keep], directed=True)


class NumpyPartition:
    def __init__(self, g, lo, hi, per_words):
        self.g, self.lo, self.hi, self.per = g, lo, hi, per_words
        self.b = O.build_bvss(rows_graph(g, lo, hi))
        self.words = (g.n + 31) // 32
        self.w_lo = lo // 32

    def row_range(self):
        return self.lo, self.hi

    def begin(self, src):
        self.L = np.full(self.g.n, INF, np.uint32)
        self.Vc = np.zeros(self.words, np.uint32)
        self.Vn = np.zeros(self.words, np.uint32)
        if self.lo <= src < self.hi:
            self.L[src] = 0
            self.Vc[src >> 5] |= np.uint32(1 << (src & 31))
            self.Vn[src >> 5] |= np.uint32(1 << (src & 31))
        ss = src >> 3
        self.queue = [(v, 1 << (src & 7)) for v in range(self.b.real_ptrs[ss], self.b.real_ptrs[ss + 1])]
        return len(self.queue)

    def pull(self):
        m = self.b.masks.reshape(-1, 32)
        r = self.b.row_ids.reshape(-1, 32, 4)
        for v, a in self.queue:
            for c in range(4):
                hit = ((m[v] >> np.uint32(8 * c)) & np.uint32(a)) != 0
                for u in r[v, hit, c]:
                    u = int(u)
                    bit = np.uint32(1 << (u & 31))
                    if not (self.Vc[u >> 5] & bit):
                        self.Vn[u >> 5] |= bit

    def sweep(self, level):
        whi = (self.hi + 31) // 32
        diff = self.Vn[self.w_lo:whi] & ~self.Vc[self.w_lo:whi]
        self.Vc[self.w_lo:whi] |= diff
        for k, d in enumerate(diff):
            d = int(d)
            while d:
                b = (d & -d).bit_length() - 1
                d &= d - 1
                self.L[32 * (self.w_lo + k) + b] = level
        out = np.zeros(self.per, np.uint32)
        out[: len(diff)] = diff
        return torch.from_numpy(out.view(np.int32).copy())

    def enqueue(self, full):
        d = full.numpy().view(np.uint32)[: self.words]
        self.queue = []
        for w in np.flatnonzero(d):
            for s in range(4):
                a = (int(d[w]) >> (8 * s)) & 0xFF
                if a:
                    ss = 4 * int(w) + s
                    self.queue += [(v, a) for v in range(self.b.real_ptrs[ss], self.b.real_ptrs[ss + 1])]
        return len(self.queue), int(sum(bin(int(x)).count("1") for x in d))

    def levels(self):
        return self.L[self.lo:self.hi].copy()
