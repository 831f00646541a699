#!/usr/bin/env python
"""Benchmark: harmonic-mean GTEPS of the fused sm_100a BFS over BLEST BVSS structures.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one BFS (init_state + every level, one fused cooperative launch) from the next
seeded source on the resident BVSS. Default workload (BASELINE.json configs[1]):
GAP-style Kronecker scale 24 (RMAT a/b/c = .57/.19/.19, edgefactor 16, GAP-style random
relabel), compression-oriented reorder (auto plan -> Jaccard windows w = 2^16), engine
policy "b200". Graph generation, reordering and BVSS construction run on the GPU before
the timed region. Inputs (3.4 GB BVSS) exceed the 126 MB L2, so no flush is needed.

Parity (default on, outside the timed region): the ORIGINAL graph is rebuilt on the host
from the generator twins (oracle/, orc_gen_csr: generate -> relabel -> from_edges), the
CPU reference BFS (orc_reference_bfs, R:src/graph.cpp:144-167) runs from every timed
source in original ids, and the GPU level arrays, mapped back through the ordering
permutation, must equal it bit for bit; the line's "parity" block reports the count.
The cpu_baseline leg's reference-engine levels are compared with the GPU levels too.

N > 1 (torchrun): every rank holds the full structure and runs its own share of the
sources (no data-path collective, "scaling": "weak"); value = sum over ranks of each
rank's harmonic-mean GTEPS, each rank timed on its device, the max elapsed over ranks
reported.

--impl reference: host CPU only — the product library is never loaded. The structure is
built by the CPU oracle (generator twins, classifier, Jaccard windows / RCM restatements,
BVSS builder; each pinned to the reference) and the UNMODIFIED reference engine
(oracle/_ref: R:src/bfs_engine.cpp run_eager/run_lazy, workers = all host threads,
num_warps = 32 x threads) is timed over it from the same sources, on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (kind, params, ordering, description)
    "c1": ("rmat", dict(scale=16, ef=16, seed=1, relabel=None), "identity",
           "RMAT scale 16 ef16 (C1), identity order"),
    "c2": ("rmat", dict(scale=24, ef=16, seed=1, relabel=2), "auto",
           "GAP-style Kronecker scale 24 ef16, random relabel, compression reorder (auto: Jaccard windows w=2^16)"),
    "c3": ("urand", dict(scale=24, ef=16, seed=3), "auto",
           "GAP-style urand scale 24 ef16, ordering as routed by the classifier"),
    "c4": ("grid", dict(rows=4096, cols=8192, relabel=4), "rcm",
           "2D 4-neighbour grid 4096x8192 (33.5M vertices), scrambled then RCM"),
    "c5": ("rmat", dict(scale=27, ef=16, seed=1, relabel=2), "auto",
           "GAP-style Kronecker scale 27 ef16"),
}


def coll_dev():
    """Device for the small bookkeeping collectives: CUDA under NCCL, host under gloo."""
    import torch.distributed as dist
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled in-process through NVML every few ms from a
    background thread (no subprocess start-up lag), started before the warm-up so it is
    sampling when the timed region begins; summary() keeps the samples taken while the
    timed region ran (mark()/unmark() bracket it), or the nearest ones when it was
    shorter than the sampling period."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.rows = []  # (host time, [sm_mhz, sm_max_mhz, reasons bitmask])
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        self.thread = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = self._handle(nv)
            self.sm_max = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: the summary says "unsampled"
            log(f"clock sampler unavailable: {e}")
            return self
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()
        while not self.rows and self.thread.is_alive():  # the first sample precedes the timed region
            time.sleep(self.period)
        return self

    def _handle(self, nv):
        # CUDA and NVML enumerate devices in the same (PCI) order when CUDA_VISIBLE_DEVICES is
        # unset, as on the bench box; the process's device index is its local rank
        return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((time.time(), [sm, self.sm_max, rs]))
            except Exception:
                return
            time.sleep(self.period)

    def mark(self):
        self.t0 = time.time()

    def unmark(self):
        self.t1 = time.time()

    def stop(self):
        self._stop.set()
        if self.thread:
            self.thread.join(timeout=1)

    def summary(self):
        rows = list(self.rows)
        if self.t0 is not None and self.t1 is not None and rows:
            inside = [r for t, r in rows if self.t0 <= t <= self.t1]
            if not inside:  # region shorter than the sampling period: the nearest samples
                mid = 0.5 * (self.t0 + self.t1)
                inside = [r for t, r in sorted(rows, key=lambda tr: abs(tr[0] - mid))[:3]]
            rows = inside
        else:
            rows = [r for _, r in rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({name for r in rows for name, bit in self.REASONS if int(r[2]) & bit})
        return {"sm_mhz": statistics.median(float(r[0]) for r in rows), "sm_max_mhz": max(float(r[1]) for r in rows),
                "reasons": reasons, "samples": len(rows), "source": "NVML in-process"}


def gpu_local_affinity(dev: int):
    """Pin this process to the CPUs of the GPU's NUMA node (NVML) so pinned host buffers
    land next to the GPU's PCIe root: the e2e level copies otherwise swing with process
    placement (C2 e2e 157 vs 89 GTEPS on the same box). Returns the previous affinity."""
    old = os.sched_getaffinity(0)
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(dev)
        words = (os.cpu_count() + 63) // 64
        mask = nv.nvmlDeviceGetCpuAffinity(h, words)
        cpus = {64 * i + b for i, w in enumerate(mask) for b in range(64) if (w >> b) & 1}
        cpus &= old
        if cpus:
            os.sched_setaffinity(0, cpus)
    except Exception:
        pass
    return old


def oracle_mod():
    """The CPU checker (oracle/): only the parity, cpu_baseline and reference legs use it."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    return O


def cpu_original_graph(config: str, threads: int):
    """The config's ORIGINAL graph (before the ordering) built on the host by the oracle's
    generator twins: the same (seed, index) -> edge functions as the device generators,
    the same relabel, then Graph::from_edges semantics (R:src/graph.cpp:33-55)."""
    O = oracle_mod()
    kind, prm, _, _ = CONFIGS[config]
    if kind == "rmat":
        n = 1 << prm["scale"]
        spec = ("rmat", prm["scale"], 0, prm["ef"] << prm["scale"], prm["seed"])
    elif kind == "urand":
        n = 1 << prm["scale"]
        spec = ("urand", n, 0, prm["ef"] * n, prm["seed"])
    else:
        n = prm["rows"] * prm["cols"]
        spec = ("grid", prm["rows"], prm["cols"], 0, 0)
    fw = O.random_relabel_mt(n, prm["relabel"], threads) if prm.get("relabel") is not None else None
    return O.gen_csr(*spec, forward=fw, threads=threads)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def engine_policy_lazy(n: int, m: int, num_vss: int) -> bool:
    """bench engine policy "b200": lazy unless the graph is low-degree (arcs/n < 8: grids,
    thousands of levels, where eager's one barrier per level wins) or small (< 2^20 VSSs,
    where lazy's fixed stage-2 cost per level dominates)."""
    return m >= 8 * max(n, 1) and num_vss >= (1 << 20)


def batch_d2h_bytes(deepest: list, n: int, packed: bool) -> int:
    """Level bytes one blest_bfs_batch call moves over PCIe (BfsEngine::run_batch, xfer.cuh):
    source k goes at the width in force when it launched (1 byte, then 2, then u32); a source
    whose deepest level does not fit is re-copied as u32 once its copy lands (two sources
    later), which also widens the sources launched after that."""
    if not packed:
        return 4 * n * len(deepest)
    width, wk, total = 1, [0] * len(deepest), 0

    def fin(j):
        nonlocal width
        if not wk[j] or deepest[j] < (255 if wk[j] == 1 else 65535):
            return 0
        if width == wk[j]:
            width = 2 if (wk[j] == 1 and deepest[j] < 65535) else 0
        return 4 * n

    for k in range(len(deepest)):
        if k >= 2:
            total += fin(k - 2)
        wk[k] = width
        total += wk[k] * n + 8 if wk[k] else 4 * n
    for j in range(max(0, len(deepest) - 2), len(deepest)):
        total += fin(j)
    return total


def prepare(config: str, ordering_override: str | None, window: int, build: bool = True):
    """Generate -> (relabel) -> plan/order -> permute -> build, all on the GPU (build=False:
    the row-partitioned mode builds one BVSS slice per rank instead)."""
    import paper_2512_21967_b200 as B
    kind, prm, ordering, desc = CONFIGS[config]
    ordering = ordering_override or ordering
    t0 = time.time()
    if kind == "rmat":
        g = B.Graph.generate_rmat(prm["scale"], prm["ef"], prm["seed"])
    elif kind == "urand":
        n = 1 << prm["scale"]
        g = B.Graph.generate_urand(n, prm["ef"] * n, prm["seed"])
    else:
        g = B.Graph.generate_grid(prm["rows"], prm["cols"])
    if prm.get("relabel") is not None:
        g = B.apply_permutation(g, B.relabel_permutation(g.num_vertices(), prm["relabel"]))
    t_gen = time.time() - t0
    t0 = time.time()
    force = {"auto": None, "identity": B.OrderingStrategy.Identity, "rcm": B.OrderingStrategy.Rcm,
             "jaccard": B.OrderingStrategy.JaccardWindows, "random": B.OrderingStrategy.Random}[ordering]
    plan = B.select_plan(g, 8, B.SelectDefaults(window_size=window, force=force))
    perm = B.make_permutation(g, plan, 8, seed=7)
    t_order = time.time() - t0
    t0 = time.time()
    gp = g if perm.is_identity() else B.apply_permutation(g, perm)
    b = None
    if build:
        b = B.build_bvss(gp)
        b.producing_permutation = perm
        b.ordering_tag = plan.strategy.value
    t_build = time.time() - t0
    return dict(g=g, gp=gp, b=b, plan=plan, perm=perm, desc=desc, ordering=ordering,
                times=dict(generate_s=round(t_gen, 3), order_s=round(t_order, 3), build_s=round(t_build, 3)))


def b_alg(n, D, P, V, L, lazy):
    """Algorithmic bytes per BFS: 648 D + 4 P + 4 n + 4 V + k (n/8) L with
    k = 2 for lazy (the V_curr + V_next word sweep of every level) and k = 0 for eager: the
    reference clears F_next (n/8 bytes) every level, the B200 eager engine never does (its
    triple-buffered frontier zeroes only the bytes the previous level set)."""
    return 648 * D + 4 * P + 4 * n + 4 * V + (2 if lazy else 0) * (n // 8) * L


def cpu_reference_sample(prep, sources_bvss, mode_lazy, budget_s, threads, max_steps, gpu_levels=None):
    """Time the reference engine (oracle/_ref) on a bounded sample of the same workload, over
    the GPU-built BVSS arrays. With gpu_levels (source -> level array, permuted ids) every
    sampled source's reference-engine levels are compared with the GPU's."""
    O = oracle_mod()
    b = prep["b"]
    rp, v2r, rows, masks = b.arrays()
    arr = O.BvssArrays(b.n, b.m, b.num_slice_sets, b.num_vss, b.num_unpadded_slices, rp, v2r, rows, masks)
    if O.ref_available():
        rb = O.ref_bvss_from_arrays(arr)
        kind = "reference"
        run = lambda s: rb.run(int(s), mode_lazy, warps=32 * threads, workers=threads,
                               want_levels=True, n=b.n, trace_cap=1 << 16)
        cores = threads
    else:
        kind = "port"
        run = lambda s: O.run_engine(arr, int(s), mode_lazy)
        cores = 1
    times, counters, checked, mism = [], [], 0, 0
    t_start = time.time()
    for s in sources_bvss[:max_steps]:
        t0 = time.perf_counter()
        r = run(s)
        times.append(time.perf_counter() - t0)
        counters.append(r.counters)
        if gpu_levels is not None and int(s) in gpu_levels:
            checked += 1
            mism += int(not np.array_equal(r.levels, gpu_levels[int(s)]))
        if time.time() - t_start > budget_s:
            break
    del arr
    return kind, cores, times, counters, dict(checked=checked, mismatches=mism)


def validate_levels(config, threads, srcs_orig, gpu_levels, fwd, edges):
    """Parity of the timed sources against the CPU reference BFS on the host-built ORIGINAL
    graph: GPU levels (permuted ids) mapped back through the ordering (levels_orig[v] =
    levels_gpu[forward[v]]) must equal orc_reference_bfs's; the traversed-edge numerator
    and the non-isolated source picks are cross-checked too."""
    O = oracle_mod()
    t0 = time.time()
    g = cpu_original_graph(config, threads)
    t_graph = time.time() - t0
    t0 = time.time()
    want, _ = O.reference_bfs_many(g, np.asarray(srcs_orig, np.uint32), threads)
    t_bfs = time.time() - t0
    mism, bad_edges = [], 0
    for k, s in enumerate(srcs_orig):
        got = gpu_levels[k] if fwd is None else gpu_levels[k][fwd]
        if not np.array_equal(got, want[k]):
            mism.append(int(s))
        if O.traversed_edges(g, want[k]) != edges[k]:
            bad_edges += 1
    return dict(checked=len(srcs_orig), mismatches=len(mism), mismatched_sources=mism[:8],
                edges_mismatches=bad_edges,
                oracle="orc_reference_bfs (R:src/graph.cpp:144-167) from the original source ids on the "
                       "host-built original graph (orc_gen_csr generator twins + relabel + from_edges); "
                       "GPU levels mapped back through the ordering permutation",
                cpu_graph_s=round(t_graph, 1), cpu_bfs_s=round(t_bfs, 1), threads=threads), g


def run_reference(args):
    """--impl reference: host CPU only, the product library is never loaded. Structure by the
    pinned CPU oracle (generator twins -> classifier -> Jaccard windows / RCM -> permute ->
    BVSS), then the UNMODIFIED reference engine (oracle/_ref, R:src/bfs_engine.cpp
    run_eager / run_lazy) timed from the same sources as our arm's rank 0."""
    O = oracle_mod()
    threads = os.cpu_count() or 1
    kind, prm, ordering, desc = CONFIGS[args.config]
    ordering = args.order or ordering
    t0 = time.time()
    g = cpu_original_graph(args.config, threads)
    t_gen = time.time() - t0
    t0 = time.time()
    n = g.n
    cls = O.classify(g)
    strategy = {"auto": "jaccard-windows" if cls["is_social_like"] else "rcm", "identity": "identity",
                "rcm": "rcm", "jaccard": "jaccard-windows"}[ordering]
    if strategy == "jaccard-windows":
        fwd = O.jaccard_windows(g, args.window, 8, threads)
    elif strategy == "rcm":
        fwd = O.rcm(g)
    else:
        fwd = None
    t_order = time.time() - t0
    t0 = time.time()
    gp = O.permute_csr(g, fwd, threads) if fwd is not None else g
    arr = O.build_bvss_mt(gp, threads)
    # the reference engine indexes slots with u32 (R:include/blest/bvss.hpp:60-62): from 2^25
    # VSSs (C5) it is invalid and the reference path is reference_bfs
    engine_ok = arr.num_vss < (1 << 25)
    rb = O.ref_bvss_from_arrays(arr) if engine_ok else None
    t_build = time.time() - t0
    lazy = engine_policy_lazy(n, arr.m, arr.num_vss) if args.mode == "b200" else (args.mode == "lazy")
    total = args.steps * max(args.gpus, 1) + args.warmup
    srcs_orig = O.pick_sources(g, total, args.source_seed)
    srcs = fwd[srcs_orig] if fwd is not None else srcs_orig
    warm, mine = srcs[: args.warmup], srcs[args.warmup: args.warmup + args.steps]
    if engine_ok:
        run = lambda s: rb.run(int(s), lazy, warps=32 * threads, workers=threads, want_levels=True, n=n,
                               trace_cap=1 << 16)
    else:
        class _R:
            pass

        def run(s):
            r = _R()
            r.levels = O.reference_bfs(gp, int(s))[0]
            return r
        del arr
    for s in warm:
        run(s)
    times, edges, t_start = [], [], time.time()
    for s in mine:
        t1 = time.perf_counter()
        r = run(s)
        times.append(time.perf_counter() - t1)
        edges.append(O.traversed_edges(gp, r.levels))
        if time.time() - t_start > 150.0:
            break
    # self-check of the timed engine against the CPU reference BFS (first source, untimed)
    want = O.reference_bfs(g, int(srcs_orig[args.warmup]))[0]
    got = run(mine[0]).levels
    ok = bool(np.array_equal(got if fwd is None else got[fwd], want))
    hm = len(times) / sum(t / e for t, e in zip(times, edges)) / 1e9
    workload = dict(workload=args.config, graph=desc, n=n, arcs=int(gp.m),
                    num_vss=int(arr.num_vss) if engine_ok else None,
                    ordering=strategy, engine="lazy" if lazy else "eager", engine_policy=args.mode,
                    sources=len(times), source_seed=args.source_seed,
                    prep_s=dict(generate_s=round(t_gen, 3), order_s=round(t_order, 3), build_s=round(t_build, 3)),
                    parallelism=f"{threads} host threads")
    cpu = dict(value=round(hm, 6), unit="GTEPS", cores=threads if engine_ok else 1,
               kind="reference" if (O.ref_available() and engine_ok) else "port",
               cpu_model=cpu_model(),
               sample=(f"{len(times)} of {args.steps} sources (bounded ~150 s) after {len(warm)} warm-up runs, "
                       f"R:src/bfs_engine.cpp run_{'lazy' if lazy else 'eager'} workers={threads} "
                       f"num_warps={32 * threads} over a BVSS built by the CPU oracle (no GPU)") if engine_ok else
                      (f"{len(times)} of {args.steps} sources: reference_bfs (R:src/graph.cpp:144-167, the "
                       f"oracle's restatement, 1 core); the reference engine is invalid at >= 2^25 VSSs"))
    line = dict(metric="GTEPS (harmonic mean over sources)", value=round(hm, 6), unit="GTEPS", n_gpus=args.gpus,
                steps=len(times), warmup=len(warm), ms_per_step=round(1e3 * sum(times) / len(times), 3),
                higher_is_better=True, scaling="weak", vs_baseline=None, dtype="u32", data="synthetic",
                impl="reference", config=workload, cpu_baseline=cpu,
                e2e=dict(value=round(hm, 6), unit="GTEPS", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                parity=dict(checked=1, mismatches=int(not ok),
                            oracle="reference engine levels vs orc_reference_bfs (first timed source)"))
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="b200", choices=["b200", "auto", "eager", "lazy"],
                    help="engine: b200 = lazy unless the graph is low-degree (arcs/n < 8, e.g. grids: "
                         "many levels, where eager's one barrier per level wins) or small (< 2^20 VSSs); auto = the reference's "
                         "rule (R:src/bfs_engine.cpp:358-362)")
    ap.add_argument("--pull", default="popc", choices=["popc", "mma"])
    ap.add_argument("--order", default=None, choices=["auto", "identity", "rcm", "jaccard", "random"])
    ap.add_argument("--window", type=int, default=1 << 16)
    ap.add_argument("--threads", type=int, default=0, help="threads per CTA (256/512/1024; 0 = default)")
    ap.add_argument("--grid-ctas", type=int, default=0, help="persistent grid size (0 = all co-resident CTAs)")
    ap.add_argument("--source-seed", type=int, default=1)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunk", type=int, default=64,
                    help="sources per blest_bfs_batch call in the e2e leg (capped by a 4.4 GB host buffer)")
    ap.add_argument("--e2e-pageable", action="store_true",
                    help="e2e output in pageable (pre-touched) host memory instead of pinned")
    ap.add_argument("--validate", type=int, default=-1,
                    help="parity: check this many timed sources against the CPU reference BFS on a host-built "
                         "original graph (-1 = all, 0 = off)")
    ap.add_argument("--partition", default=None, choices=["replicas", "rows"],
                    help="N>1: rows (default: one BFS row-partitioned over the ranks, SURVEY 8(e)) or "
                         "replicas (every rank holds the whole structure and runs its share of the sources)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="rows mode: nccl = one launch per level + ncclAllGather of the frontier words; "
                         "p2p = one launch per BFS, frontier words stored into the peers' buffers over "
                         "CUDA IPC (NVLink) with an in-kernel cross-rank barrier")
    ap.add_argument("--virtual-ranks", type=int, default=0,
                    help="rows partition emulated on one GPU with this many ranks (p2p exchange in one launch)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:  # rank 0 alone runs it; the other ranks exit without work
            run_reference(args)
        return

    import torch
    import torch.distributed as dist
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL over NVLink, one GPU per rank. BLEST_DIST_BACKEND=gloo lets several ranks share
        # one GPU (local % device_count) to exercise this path on a single-GPU box.
        backend = os.environ.get("BLEST_DIST_BACKEND", "nccl")
        local = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    all_cpus = gpu_local_affinity(local)
    import paper_2512_21967_b200 as B
    from paper_2512_21967_b200 import _lib as L
    lib = L.lib()
    stream = torch.cuda.current_stream()
    L.check(lib.blest_set_stream(C.c_void_p(stream.cuda_stream)))

    if args.partition is None:
        args.partition = "rows" if world > 1 else "replicas"
    rows_mode = args.partition == "rows" or args.virtual_ranks > 0
    prep = prepare(args.config, args.order, args.window, build=not rows_mode)
    g, b, plan, perm = prep["g"], prep["b"], prep["plan"], prep["perm"]
    if rows_mode:
        run_partitioned(args, prep, B, L, lib, perm, world, rank, local, stream)
        if world > 1:
            dist.destroy_process_group()
        return
    if args.mode == "b200":
        # measured: lazy wins on large Kron and urand (C3 2.7 vs 4.75 ms), eager on grids (many
        # levels) and on small graphs, where lazy's ~15 µs fixed stage-2 cost per level
        # dominates (C1 RMAT-16: eager 0.091 vs lazy 0.218 ms per BFS)
        mode = B.EngineMode.Lazy if engine_policy_lazy(b.n, b.m, b.num_vss) else B.EngineMode.Eager
    else:
        cfg = B.EngineConfig(mode=B.engine_mode_from_string(args.mode), pull=args.pull)
        mode = B.choose_mode(b, plan, cfg)
    lazy = mode == B.EngineMode.Lazy
    n = b.n
    total_sources = args.steps * world + args.warmup
    srcs_orig = g.pick_sources(total_sources, args.source_seed)
    srcs = perm.forward_map()[srcs_orig] if not perm.is_identity() else srcs_orig
    mine = srcs[args.warmup + rank * args.steps: args.warmup + (rank + 1) * args.steps]
    warm = srcs[: args.warmup]
    threads = os.cpu_count() or 1
    workload = dict(workload=args.config, graph=prep["desc"], n=n, arcs=int(b.m),
                    num_vss=int(b.num_vss), ordering=plan.strategy.value, engine=mode.value, engine_policy=args.mode,
                    pull=args.pull, sources=len(mine) * world, source_seed=args.source_seed,
                    l2=("inputs larger than L2 (BVSS %.2f GB > 126 MB), no flush" % (b.num_vss * 644 / 1e9)
                        if b.num_vss * 644 >= 2 * 126e6 else
                        "BVSS %.1f MB fits in L2: 512 MB L2 flush before every timed BFS" % (b.num_vss * 644 / 1e6)),
                    prep_s=prep["times"], parallelism=f"source-sharded x{world}" if world > 1 else "1 GPU")

    ecfg = L.EngineConfigT(L.MODE_LAZY if lazy else L.MODE_EAGER,
                           L.PULL_MMA if args.pull == "mma" else L.PULL_POPC, 0, 0, args.grid_ctas, args.threads)
    ctr = L.CountersT()
    # ---- engine preparation (lazy: the hot-row view), timed and sized apart from the BFS ----
    t0 = time.time()
    ebytes = C.c_uint64()
    L.check(lib.blest_bfs_prepare(b.handle, C.byref(ecfg), C.byref(ebytes)))
    prep["times"]["engine_prepare_s"] = round(time.time() - t0, 3)
    workload["engine_device_bytes"] = int(ebytes.value)
    workload["bvss_device_bytes"] = int(4 * (b.num_slice_sets + 1) + 4 * b.num_vss + 4 * 128 * b.num_vss
                                        + 4 * 32 * b.num_vss)
    # ---- census (untimed): deterministic counters + traversed edges (+ levels) per source ----
    nval = len(mine) if args.validate < 0 else min(args.validate, len(mine))
    if world > 1 and rank != 0:
        nval = 0  # replicas run the same code path: rank 0 validates its share
    keep = {int(s) for s in mine[:max(nval, 8)]}
    census = census_of(lib, L, b, prep, mine, lazy, args.pull, args.threads, args.grid_ctas, keep_levels=keep)
    parity = None
    if nval:
        fm = None if perm.is_identity() else perm.forward_map()
        srcs_mine_orig = srcs_orig[args.warmup + rank * args.steps: args.warmup + rank * args.steps + nval]
        parity, gcpu = validate_levels(args.config, threads, srcs_mine_orig,
                                       [census[k]["levels"] for k in range(nval)], fm,
                                       [census[k]["E"] for k in range(nval)])
        O = oracle_mod()
        parity["source_picks_match"] = bool(np.array_equal(O.pick_sources(gcpu, total_sources, args.source_seed),
                                                           srcs_orig))
        del gcpu
        log(f"parity: {parity['checked']} sources, {parity['mismatches']} mismatches "
            f"(cpu graph {parity['cpu_graph_s']} s, cpu bfs {parity['cpu_bfs_s']} s)")
    # ---- warmup (the clock sampler starts here so it is running in the timed region) ----
    clk = ClockSampler(local).start()
    for s in warm:
        L.check(lib.blest_bfs(b.handle, int(s), C.byref(ecfg), None, C.byref(ctr), None, 0))
    # ---- timed region: K fused launches, CUDA events on the launching stream ----
    # Structures smaller than 2x the 126 MB L2 (C1) get an L2 flush (a 512 MB write) before
    # every timed BFS, outside its event pair; larger ones stream from HBM anyway.
    flush = b.num_vss * 644 < 2 * 126e6
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if flush else None
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(len(mine))]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(len(mine))]
    launches0 = lib.blest_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.mark()
    for k, s in enumerate(mine):
        if flush:
            scratch.fill_(k & 0xFF)
        ev_s[k].record(stream)
        L.check(lib.blest_bfs_launch(b.handle, int(s), C.byref(ecfg)))
        ev_e[k].record(stream)
    torch.cuda.synchronize()
    clk.unmark()
    clk.stop()
    if world > 1:
        dist.barrier()
    launches = lib.blest_kernel_launches() - launches0
    g_ctas, g_thr = C.c_uint32(), C.c_uint32()
    L.check(lib.blest_bfs_last_geometry(b.handle, C.byref(g_ctas), C.byref(g_thr)))
    L.check(lib.blest_bfs_finish(b.handle, None, C.byref(ctr), None, 0))
    t = np.array([ev_s[k].elapsed_time(ev_e[k]) / 1e3 for k in range(len(mine))])
    E = np.array([c["E"] for c in census], np.float64)
    hm = len(t) / float(np.sum(t / E)) / 1e9
    total_s = float(t.sum())
    balg = np.array([b_alg(n, c["D"] - c["U"], c["P"], c["V"], c["L"] - (1 if c["U"] else 0), lazy)
                     for c in census], np.float64)
    achieved = float(np.sum(balg) / total_s / 1e9)
    # the same formula on the counters alone (SURVEY 8(d) reads D off the reference's counters,
    # which include a barren last level the engines account without streaming it)
    balg_ctr = np.array([b_alg(n, c["D"], c["P"], c["V"], c["L"], lazy) for c in census], np.float64)
    achieved_ctr = float(np.sum(balg_ctr) / total_s / 1e9)
    peak, peak_kind = load_peaks()
    value, elapsed = hm, total_s
    if world > 1:
        tt = torch.tensor([hm, total_s], dtype=torch.float64, device=coll_dev())
        allv = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(allv, tt)
        value = float(sum(x[0].item() for x in allv))
        elapsed = float(max(x[1].item() for x in allv))

    # ---- e2e through the C-ABI with host buffers (pinned) ----
    # blest_bfs_batch: the public many-sources call (the CLI's loop over its sources as one
    # call); source k's level array crosses PCIe narrowed and is widened into the host buffer
    # while source k+1 runs. One call for all sources up to a 4.4 GB host buffer (C2: 64, C5:
    # 8; chunks of 16 measured 160 vs 169 GTEPS on C2 — each call ends with one exposed copy,
    # profiles/r02_e2e_ab/); each source's time = its call's wall time / size.
    e2e = None
    if not args.no_e2e:
        chunk = max(1, min(args.e2e_chunk, len(mine), int(4.4e9 // (4 * max(n, 1)))))
        if args.e2e_pageable:  # pre-touched, so no first-touch page faults in the timed calls
            hl = torch.ones((chunk, n), dtype=torch.int32)
        else:
            hl = torch.empty((chunk, n), dtype=torch.int32, pin_memory=True)
        hsrc = torch.empty(chunk, dtype=torch.int32, pin_memory=True)
        cbuf = (L.CountersT * chunk)()
        torch.cuda.synchronize()
        te = np.zeros(len(mine))
        d2h = 0  # level bytes over PCIe, per blest_bfs_batch's width rule (xfer.cuh)
        packed = os.environ.get("BLEST_D2H_PACK", "1") != "0"
        for c0 in range(0, len(mine), chunk):
            part = np.ascontiguousarray(mine[c0:c0 + chunk], np.uint32)
            t0 = time.perf_counter()
            hsrc.numpy().view(np.uint32)[: len(part)] = part
            L.check(lib.blest_bfs_batch(b.handle, C.c_void_p(hsrc.data_ptr()), len(part), C.byref(ecfg),
                                        C.c_void_p(hl.data_ptr()), C.cast(cbuf, C.c_void_p)))
            te[c0:c0 + len(part)] = (time.perf_counter() - t0) / len(part)
            d2h += batch_d2h_bytes([c.levels_processed for c in list(cbuf)[: len(part)]], n, packed)
        e2e_hm = len(te) / float(np.sum(te / E)) / 1e9
        e2e = dict(value=round(e2e_hm * world, 4), unit="GTEPS", h2d_bytes_per_step=4,
                   d2h_bytes_per_step=int(d2h / len(mine)) + 8 * 8 + 16,
                   note=f"blest_bfs_batch() in chunks of {chunk} sources: source ids in, every source's full "
                        f"u32 level array ({'pageable' if args.e2e_pageable else 'pinned'} host) + counters out, host wall clock per chunk / chunk size; "
                        + ("levels cross PCIe as (level+1) in 1-2 bytes and host threads widen them to u32 "
                           "inside the call" if packed else "levels cross PCIe as u32 (BLEST_D2H_PACK=0)"))

    # ---- CPU baseline (rank 0, N = 1 only): every host core again ----
    os.sched_setaffinity(0, all_cpus)
    cpu = None
    # The reference engine indexes slots with u32 (R:include/blest/bvss.hpp:60-62) and is
    # invalid from 2^25 VSSs (C5); there the baseline is reference_bfs alone.
    engine_ok = b.num_vss < (1 << 25)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        echeck = None
        if engine_ok:
            glv = {int(mine[k]): census[k]["levels"] for k in range(len(mine)) if census[k].get("levels") is not None}
            kind, cores, ctimes, _, echeck = cpu_reference_sample(prep, mine, lazy, args.cpu_budget, threads,
                                                                  max_steps=8, gpu_levels=glv)
            chm = len(ctimes) / sum(tc / e for tc, e in zip(ctimes, E[: len(ctimes)])) / 1e9
            cpu = dict(value=round(chm, 6), unit="GTEPS", cores=cores, kind=kind, cpu_model=cpu_model(),
                       sample=f"first {len(ctimes)} of the {len(mine)} timed sources (~{args.cpu_budget:.0f} s "
                              f"budget), run_{'lazy' if lazy else 'eager'} over the same BVSS arrays",
                       engine_levels_vs_gpu=echeck)
        else:
            cpu = dict(value=None, unit="GTEPS", cores=1, kind="port", cpu_model=cpu_model(),
                       sample="reference engine not run: its u32 slot index wraps at >= 2^25 VSSs "
                              f"({b.num_vss} here, R:include/blest/bvss.hpp:60-62); reference_bfs below")
        # reference_bfs on one core (R:src/graph.cpp:144-167, the oracle's restatement), one source
        O = oracle_mod()
        g1 = O.Csr(n, *prep["gp"].csr())
        t1 = time.perf_counter()
        lv1 = O.reference_bfs(g1, int(mine[0]))[0]
        t1 = time.perf_counter() - t1
        cpu["reference_bfs_1core"] = dict(value=round(census[0]["E"] / t1 / 1e9, 6), unit="GTEPS", cores=1,
                                          kind="port", seconds=round(t1, 3),
                                          levels_match_gpu=bool(census[0].get("levels") is None or
                                                                np.array_equal(lv1, census[0]["levels"])),
                                          sample="first timed source, orc_reference_bfs (FIFO queue BFS)")
        if cpu["value"] is None:
            cpu["value"] = cpu["reference_bfs_1core"]["value"]
        if parity is not None and echeck is not None:
            parity["engine_levels_vs_gpu"] = echeck
        del g1

    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tp):
        tj = json.load(open(tp))
        if tj.get("engine") == mode.value and tj.get("pull") == args.pull:
            traffic = tj.get("dram_bytes_per_launch")
    if rank == 0:
        line = dict(
            metric="GTEPS (harmonic mean over sources)", value=round(value, 4), unit="GTEPS", n_gpus=world,
            steps=len(mine), warmup=len(warm), ms_per_step=round(1e3 * elapsed / len(mine), 4),
            higher_is_better=True, scaling="weak", vs_baseline=None, dtype="u32", data="synthetic",
            config=workload,
            roofline=dict(bound="hbm", achieved=round(achieved, 1), peak=peak, unit="GB/s",
                          frac=round(achieved / peak, 4), traffic=traffic,
                          peak_source=f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind == "measured" else "fallback 6.65 TB/s",
                          algorithmic_bytes_per_bfs=int(np.mean(balg)),
                          formula="648 D + 4 P + 4 n + 4 V + k (n/8) L (SURVEY 8(d)); D and L without a "
                                  "barren last level the engine did not pull (detail.mean_unpulled)",
                          frac_counter_bytes=round(achieved_ctr / peak, 4),
                          frac_counter_bytes_note="the same formula with D and L straight from the counters "
                                                  "(the unpulled barren level counted as streamed); equals frac "
                                                  "when nothing was left unpulled"),
            cpu_baseline=cpu, e2e=e2e, gpu_launches=int(launches), parity=parity,
            clocks=clk.summary(),
            detail=dict(grid=[g_ctas.value, g_thr.value], hm_gteps_rank0=round(hm, 4), mean_ms=round(1e3 * float(t.mean()), 4),
                        min_ms=round(1e3 * float(t.min()), 4), max_ms=round(1e3 * float(t.max()), 4),
                        mean_dequeues=int(np.mean([c["D"] for c in census])),
                        mean_unpulled=int(np.mean([c["U"] for c in census])),
                        mean_levels=float(np.mean([c["L"] for c in census])),
                        mean_traversed_edges=int(E.mean()), arcs_per_s_G=round(2 * hm, 4)))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_partitioned(args, prep, B, L, lib, perm, world, rank, local, stream):
    """Row-partitioned BFS (csrc/rows.cu): rank g owns a slice-balanced range
    of destination rows and the BVSS of A[rows_g, all columns], built on its own GPU. Each
    step = one BFS from the next source over all ranks (strong scaling); value = harmonic-
    mean GTEPS of the distributed BFS, each BFS timed with CUDA events on every rank's
    stream, max over ranks. --exchange nccl: one launch per level + ncclAllGather of the
    n/8-byte frontier (host never waits on a level); p2p: one launch per BFS, peer stores
    over CUDA IPC; --virtual-ranks G: G ranks of this GPU in one launch (p2p protocol)."""
    import torch
    import torch.distributed as dist
    from paper_2512_21967_b200 import multigpu as MG
    gp = prep["gp"]
    n = gp.num_vertices()
    deg = gp.out_degrees().astype(np.int64)
    total = args.steps * 1 + args.warmup
    srcs_orig = gp.pick_sources(total, args.source_seed) if perm.is_identity() else \
        prep["g"].pick_sources(total, args.source_seed)
    srcs = perm.forward_map()[srcs_orig] if not perm.is_identity() else srcs_orig
    warm, steps = srcs[: args.warmup], srcs[args.warmup: args.warmup + args.steps]
    virtual = args.virtual_ranks > 0
    G = args.virtual_ranks if virtual else world
    t0 = time.time()
    bounds, slices = MG.partition_rows(gp, G)
    t_part = time.time() - t0
    t0 = time.time()
    if virtual:
        engs = [MG.RowsEngine(gp, r, G, bounds) for r in range(G)]
        MG.set_local_peers(engs)
        mode = f"rows x{G} virtual ranks on 1 GPU (p2p exchange protocol, one launch per BFS)"

        def run(s):
            MG.group_bfs(engs, int(s))

        def results(levels):
            return [e.finish(levels) for e in engs]
    else:
        eng = MG.RowsEngine(gp, rank, G, bounds)
        engs = [eng]
        if args.exchange == "p2p":
            MG.exchange_ipc_handles(eng)
            mode = f"rows x{G} ranks, p2p: frontier words stored into peers over CUDA IPC, one launch per BFS"

            def run(s):
                eng.bfs(int(s))
        else:
            stepper = MG.SteppedBfs(eng, MG.torch_allgather(), ahead=2)
            mode = f"rows x{G} ranks, {dist.get_backend().upper()} all-gather of the frontier per level"

            def run(s):
                stepper.run(int(s), levels=False)

        def results(levels):
            return [eng.finish(levels)]
    torch.cuda.synchronize()
    t_build = time.time() - t0
    arcs = int(gp.num_edges())
    del prep["gp"]
    vss = [e.num_vss for e in engs]
    if not virtual and world > 1:
        tv = torch.tensor([float(v) for v in vss], dtype=torch.float64, device=coll_dev())
        allv = [torch.zeros_like(tv) for _ in range(world)]
        dist.all_gather(allv, tv)
        vss = [int(x.item()) for x in allv]

    def sync_all():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for s in warm:
        run(s)
        results(False)
    clk = ClockSampler(local).start()
    launches0 = lib.blest_kernel_launches()
    times, edges, queues, iters = [], [], [], []
    for s in steps:
        sync_all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if rank == 0:
            clk.mark()
        e0.record(stream)
        run(s)
        e1.record(stream)
        torch.cuda.synchronize()
        if rank == 0:
            clk.unmark()
        res = results(True)
        t = e0.elapsed_time(e1) / 1e3
        e = sum(int(deg[r.row_lo:r.row_hi][r.levels != 0xFFFFFFFF].sum()) for r in res)
        q = sum(r.queue - r.unpulled for r in res)  # VSSs actually pulled (exhaustion exit)
        if world > 1 and not virtual:
            tt = torch.tensor([t, float(e), float(q)], dtype=torch.float64, device=coll_dev())
            tmax = tt.clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            dist.all_reduce(tt, op=dist.ReduceOp.SUM)
            t, e, q = float(tmax[0].item()), int(tt[1].item()), int(tt[2].item())
        times.append(t)
        edges.append(e // 2)
        queues.append(q)
        iters.append(res[0].iterations)
    clk.stop()
    launches = lib.blest_kernel_launches() - launches0
    t = np.array(times)
    E = np.array(edges, np.float64)
    hm = len(t) / float(np.sum(t / E)) / 1e9

    # ---- e2e: the public call per BFS with the owned levels copied to host, wall clock ----
    te = []
    for s in steps[: min(8, len(steps))]:
        sync_all()
        w0 = time.perf_counter()
        run(s)
        results(True)
        w = time.perf_counter() - w0
        if world > 1 and not virtual:
            tw = torch.tensor([w], dtype=torch.float64, device=coll_dev())
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
            w = float(tw.item())
        te.append(w)
    te = np.array(te)
    e2e_hm = len(te) / float(np.sum(te / E[: len(te)])) / 1e9

    # ---- parity: assembled levels of the first timed sources vs the CPU reference BFS ----
    parity = None
    nval = len(steps) if args.validate < 0 else min(args.validate, len(steps))
    nval = min(nval, 8)
    if nval:
        gathered = []
        for s in steps[:nval]:
            run(s)
            res = results(True)
            if virtual:
                gathered.append(MG.assemble(res, n))
            else:
                r = res[0]
                per_rows = 32 * max(b - a for a, b in zip(bounds, bounds[1:]))
                mine = torch.full((per_rows,), -1, dtype=torch.int64, device=coll_dev())
                mine[: r.row_hi - r.row_lo] = torch.from_numpy(r.levels.astype(np.int64)).to(coll_dev())
                parts = [torch.empty_like(mine) for _ in range(world)]
                dist.all_gather(parts, mine)
                if rank == 0:
                    full = np.concatenate([p.cpu().numpy()[: min(32 * bounds[i + 1], n) - min(32 * bounds[i], n)]
                                           for i, p in enumerate(parts)])
                    gathered.append(full.astype(np.uint32))
        if rank == 0:
            fm = None if perm.is_identity() else perm.forward_map()
            parity, gcpu = validate_levels(args.config, os.cpu_count() or 1, srcs_orig[args.warmup: args.warmup + nval],
                                           gathered, fm, edges[:nval])
            del gcpu
            log(f"parity (rows x{G}): {parity['checked']} sources, {parity['mismatches']} mismatches")
    if rank == 0:
        peak, peak_kind = load_peaks()
        stream_b = 648.0 * float(np.mean(queues))
        achieved = stream_b / float(t.mean()) / 1e9 / G
        workload = dict(workload=args.config, graph=prep["desc"], n=n, arcs=arcs,
                        ordering=prep["plan"].strategy.value, engine="lazy (row-partitioned)",
                        partition=dict(ranks=G, word_bounds=[int(x) for x in bounds], slices=[int(x) for x in slices],
                                       vss=vss, balance="BVSS slice count (blest_partition_rows)"),
                        exchange="p2p" if (virtual or args.exchange == "p2p") else "nccl",
                        sources=len(steps), source_seed=args.source_seed,
                        prep_s=dict(prep["times"], partition_s=round(t_part, 3), rank_build_s=round(t_build, 3)),
                        parallelism=mode,
                        l2="inputs larger than L2 (BVSS slices >> 126 MB), no flush" if sum(vss) * 644 > 2 * 126e6
                        else "structure fits in L2 (no flush in rows mode)")
        line = dict(metric="GTEPS (harmonic mean over sources)", value=round(hm, 4), unit="GTEPS", n_gpus=world,
                    steps=len(t), warmup=len(warm), ms_per_step=round(1e3 * float(t.mean()), 4),
                    higher_is_better=True, scaling="strong", vs_baseline=None, dtype="u32", data="synthetic",
                    config=workload,
                    roofline=dict(bound="hbm", achieved=round(achieved, 1), peak=peak, unit="GB/s",
                                  frac=round(achieved / peak, 4), traffic=None,
                                  peak_source=f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs), per GPU",
                                  formula="648 B x (sum over ranks of the local VSS queue) / time / GPUs: the "
                                          "stage-1 BVSS stream per GPU"),
                    e2e=dict(value=round(e2e_hm, 4), unit="GTEPS", h2d_bytes_per_step=4,
                             d2h_bytes_per_step=int(4 * n),
                             note="the public call per BFS (launches + exchange) and every rank's owned levels "
                                  "copied to host, wall clock, max over ranks"),
                    gpu_launches=int(launches), parity=parity, clocks=clk.summary(),
                    detail=dict(mean_levels=float(np.mean(iters)), mean_traversed_edges=int(E.mean()),
                                mean_local_queue_sum=int(np.mean(queues)),
                                min_ms=round(1e3 * float(t.min()), 4), max_ms=round(1e3 * float(t.max()), 4)))
        print(json.dumps(line), flush=True)


def census_of(lib, L, b, prep, sources, lazy, pull, threads=0, grid_ctas=0, keep_levels=()):
    """Per source: VSS dequeues D, pushes P, visited V, level iterations L and traversed
    undirected edges E (on the permuted graph, whose ids the level array uses); the level
    array itself (host copy, permuted ids) for the sources in keep_levels."""
    ecfg = L.EngineConfigT(L.MODE_LAZY if lazy else L.MODE_EAGER,
                           L.PULL_MMA if pull == "mma" else L.PULL_POPC, 0, 0, grid_ctas, threads)
    ctr = L.CountersT()
    lv_ptr = C.c_void_p()
    out = []
    for s in sources:
        lv = np.empty(b.n, np.uint32) if int(s) in keep_levels else None
        L.check(lib.blest_bfs(b.handle, int(s), C.byref(ecfg), lv.ctypes.data if lv is not None else None,
                              C.byref(ctr), None, 0))
        L.check(lib.blest_bfs_levels_device(b.handle, C.byref(lv_ptr)))
        unp = C.c_uint64(0)
        if hasattr(lib, "blest_bfs_last_unpulled"):  # absent only in an older BLEST_LIB experiment build
            L.check(lib.blest_bfs_last_unpulled(b.handle, C.byref(unp)))
        e = prep["gp"].traversed_edges(lv_ptr.value)
        # roofline bytes count the VSSs actually pulled: a barren last level the lazy engine
        # proved barren (every vertex with an in-edge visited) is in D but was never streamed
        out.append(dict(D=ctr.vss_dequeues, U=int(unp.value), P=ctr.queue_pushes, V=ctr.visited_count,
                        L=ctr.trace_len, E=e, levels=lv))
    return out


if __name__ == "__main__":
    main()
