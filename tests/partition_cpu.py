"""TEST INFRASTRUCTURE: a numpy backend of the row-partitioned BFS in stepped mode
(paper_2512_21967_b200/multigpu.py SteppedBfs; csrc/rows.cu k_bfs_rows<STEPPED>), built on
the oracle's BVSS builder over the row-filtered graph. Same step semantics as the GPU
engine: step(1) initialises and runs level 1; step(l > 1) unpacks the gathered frontier,
stops if it is empty (done = l - 1), else runs level l; every level ends with the owned
diff words in the send buffer. Used by the gloo (CPU, world_size 2/3) protocol tests."""
import numpy as np
import torch

import oracle as O

INF = 0xFFFFFFFF


def rows_graph(g, lo, hi):
    """Arcs of g whose target lies in [lo, hi) (the rank's slice of A)."""
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.offsets).astype(np.int64))
    keep = (g.targets >= lo) & (g.targets < hi)
    return O.from_edges(g.n, src[keep], g.targets[keep], directed=True)


class NumpyRows:
    def __init__(self, g, rank, bounds):
        self.g, self.rank, self.bounds = g, rank, list(bounds)
        self.world = len(bounds) - 1
        self.w_lo, self.w_hi = bounds[rank], bounds[rank + 1]
        self.row_lo, self.row_hi = min(32 * self.w_lo, g.n), min(32 * self.w_hi, g.n)
        self.per = max(1, max(b - a for a, b in zip(bounds, bounds[1:])))
        self.b = O.build_bvss(rows_graph(g, self.row_lo, self.row_hi))
        self.words = (g.n + 31) // 32
        self._send = torch.zeros(self.per, dtype=torch.int32)
        self.progress = self.done = self.status = 0

    def send(self):
        return self._send

    def flags(self):
        return self.progress, self.done, self.status

    def _queue(self, F):
        q = []
        for w in np.flatnonzero(F):
            for s in range(4):
                a = (int(F[w]) >> (8 * s)) & 0xFF
                if a:
                    ss = 4 * int(w) + s
                    q += [(v, a) for v in range(self.b.real_ptrs[ss], self.b.real_ptrs[ss + 1])]
        return q

    def step(self, level, src, recv):
        if level > 1 and self.done:
            return  # no-op past the end
        self.progress = level
        if level == 1:
            self.done = self.status = 0
            self.L = np.full(self.g.n, INF, np.uint32)
            self.Vc = np.zeros(self.words, np.uint32)
            self.Vn = np.zeros(self.words, np.uint32)
            if self.row_lo <= src < self.row_hi:
                self.L[src] = 0
                self.Vc[src >> 5] |= np.uint32(1 << (src & 31))
                self.Vn[src >> 5] |= np.uint32(1 << (src & 31))
            F = np.zeros(self.words, np.uint32)
            F[src >> 5] = np.uint32(1 << (src & 31))
            self.queue_total = 0
        else:
            rv = recv.numpy().view(np.uint32)
            F = np.concatenate([rv[r * self.per: r * self.per + (self.bounds[r + 1] - self.bounds[r])]
                                for r in range(self.world)])
            if not F.any():
                self.done = level - 1
                return
        # stage 1 over the local queue (lazy pull: test V_next, mark V_next)
        m = self.b.masks.reshape(-1, 32)
        rws = self.b.row_ids.reshape(-1, 32, 4)
        q = self._queue(F)
        self.queue_total += len(q)
        for v, a in q:
            for c in range(4):
                hit = ((m[v] >> np.uint32(8 * c)) & np.uint32(a)) != 0
                for u in rws[v, hit, c]:
                    u = int(u)
                    self.Vn[u >> 5] |= np.uint32(1 << (u & 31))
        # stage 2a: owned words
        diff = self.Vn[self.w_lo:self.w_hi] & ~self.Vc[self.w_lo:self.w_hi]
        self.Vc[self.w_lo:self.w_hi] |= diff
        for k, d in enumerate(diff):
            d = int(d)
            while d:
                b = (d & -d).bit_length() - 1
                d &= d - 1
                self.L[32 * (self.w_lo + k) + b] = level
        out = np.zeros(self.per, np.uint32)
        out[: len(diff)] = diff
        self._send = torch.from_numpy(out.view(np.int32).copy())

    def finish(self, levels=True):
        from paper_2512_21967_b200.multigpu import RowsResult
        lv = self.L[self.row_lo:self.row_hi].copy()
        disc = int(np.count_nonzero((lv != INF) & (lv != 0)))
        return RowsResult(lv, self.row_lo, self.row_hi, self.done, disc, self.queue_total)
