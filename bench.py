#!/usr/bin/env python
"""Benchmark: harmonic-mean GTEPS of the fused sm_100a BFS over BLEST BVSS structures.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one BFS (init_state + every level, one fused cooperative launch) from the next
seeded source on the resident BVSS. Default workload (BASELINE.json configs[1]):
GAP-style Kronecker scale 24 (RMAT a/b/c = .57/.19/.19, edgefactor 16, GAP-style random
relabel), compression-oriented reorder (auto plan -> Jaccard windows w = 2^16), auto
engine choice. Graph generation, reordering and BVSS construction run on the GPU before
the timed region. Inputs (3.4 GB BVSS) exceed the 126 MB L2, so no flush is needed.

N > 1 (torchrun): every rank holds the full structure and runs its own share of the
sources (no data-path collective, "scaling": "weak"); value = sum over ranks of each
rank's harmonic-mean GTEPS, each rank timed on its device, the max elapsed over ranks
reported.

--impl reference: the UNMODIFIED reference engine (oracle/_ref: R:src/bfs_engine.cpp
run_eager/run_lazy, with workers = all host threads, num_warps = 32 x threads) over the
same BVSS arrays and sources, on a bounded sample of steps.
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
    """nvidia-smi clocks + throttle reasons, sampled every 20 ms from before the timed region
    (nvidia-smi needs ~0.1 s to start); summary() keeps the samples read while the timed
    region ran (mark()/unmark() bracket it), or the nearest ones when it was shorter."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (host time, fields)
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def mark(self):
        self.t0 = time.time()

    def unmark(self):
        self.t1 = time.time()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append((time.time(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = self.rows
        if self.t0 is not None and self.t1 is not None and rows:
            inside = [r for t, r in rows if self.t0 <= t <= self.t1 + 0.05]
            if not inside:  # region shorter than the sampling period: the nearest samples
                mid = 0.5 * (self.t0 + self.t1)
                inside = [r for t, r in sorted(rows, key=lambda tr: abs(tr[0] - mid))[:3]]
            rows = inside
        else:
            rows = [r for _, r in rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def prepare(config: str, ordering_override: str | None, window: int, prepass: str = "none",
            postpass: str = "none"):
    """Generate -> (relabel) -> plan/order -> permute -> build, all on the GPU."""
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
    pre = B.PrePass.DegreeSort if prepass == "degree" else B.PrePass.None_
    plan = B.select_plan(g, 8, B.SelectDefaults(window_size=window, force=force, pre_pass=pre))
    perm = B.make_permutation(g, plan, 8, seed=7)
    if postpass == "hub-blocks":
        perm = B.api.hub_blocks(g, perm)
    t_order = time.time() - t0
    t0 = time.time()
    gp = g if perm.is_identity() else B.apply_permutation(g, perm)
    b = B.build_bvss(gp)
    b.producing_permutation = perm
    b.ordering_tag = plan.strategy.value
    t_build = time.time() - t0
    return dict(g=g, gp=gp, b=b, plan=plan, perm=perm, desc=desc, ordering=ordering,
                times=dict(generate_s=round(t_gen, 3), order_s=round(t_order, 3), build_s=round(t_build, 3)))


def b_alg(n, D, P, V, L, lazy):
    """Algorithmic bytes per BFS: 648 D + 4 P + 4 n + 4 V + k (n/8) L."""
    return 648 * D + 4 * P + 4 * n + 4 * V + (2 if lazy else 1) * (n // 8) * L


def cpu_reference_sample(prep, sources_bvss, mode_lazy, budget_s, threads, max_steps):
    """Time the reference engine (oracle/_ref) on a bounded sample of the same workload."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    b = prep["b"]
    rp, v2r, rows, masks = b.arrays()
    arr = O.BvssArrays(b.n, b.m, b.num_slice_sets, b.num_vss, b.num_unpadded_slices, rp, v2r, rows, masks)
    if O.ref_available():
        rb = O.ref_bvss_from_arrays(arr)
        kind = "reference"
        run = lambda s: rb.run(int(s), mode_lazy, warps=32 * threads, workers=threads,
                               want_levels=False, n=b.n, trace_cap=1 << 16)
        cores = threads
    else:
        kind = "port"
        run = lambda s: O.run_engine(arr, int(s), mode_lazy)
        cores = 1
    times, counters = [], []
    t_start = time.time()
    for s in sources_bvss[:max_steps]:
        t0 = time.perf_counter()
        r = run(s)
        times.append(time.perf_counter() - t0)
        counters.append(r.counters)
        if time.time() - t_start > budget_s:
            break
    del arr
    return kind, cores, times, counters


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
    ap.add_argument("--prepass", default="none", choices=["none", "degree"])
    ap.add_argument("--postpass", default="none", choices=["none", "hub-blocks"])
    ap.add_argument("--threads", type=int, default=0, help="threads per CTA (256/512/1024; 0 = default)")
    ap.add_argument("--grid-ctas", type=int, default=0, help="persistent grid size (0 = all co-resident CTAs)")
    ap.add_argument("--source-seed", type=int, default=1)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--validate", type=int, default=0, help="check this many sources against the CPU oracle")
    ap.add_argument("--partition", default="replicas", choices=["replicas", "rows"],
                    help="N>1: source-sharded replicas (default) or one BFS row-partitioned over the ranks")
    ap.add_argument("--virtual-ranks", type=int, default=0,
                    help="rows partition emulated on one GPU with this many ranks (lock-step, device concat)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return  # the reference arm runs on rank 0 only, the other ranks exit without work
        world = 1  # ... and without a process group (nobody else would join it)

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
    import paper_2512_21967_b200 as B
    from paper_2512_21967_b200 import _lib as L
    lib = L.lib()
    stream = torch.cuda.current_stream()
    L.check(lib.blest_set_stream(C.c_void_p(stream.cuda_stream)))

    prep = prepare(args.config, args.order, args.window, args.prepass, args.postpass)
    g, b, plan, perm = prep["g"], prep["b"], prep["plan"], prep["perm"]
    if args.mode == "b200":
        # measured: lazy wins on large Kron and urand (C3 2.7 vs 4.75 ms), eager on grids (many
        # levels) and on small graphs, where lazy's ~15 µs fixed stage-2 cost per level
        # dominates (C1 RMAT-16: eager 0.091 vs lazy 0.218 ms per BFS)
        mode = B.EngineMode.Lazy if (b.m >= 8 * max(b.n, 1) and b.num_vss >= (1 << 20)) else B.EngineMode.Eager
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
                    pull=args.pull, prepass=args.prepass, postpass=args.postpass, sources=len(mine) * world, source_seed=args.source_seed,
                    l2=("inputs larger than L2 (BVSS %.2f GB > 126 MB), no flush" % (b.num_vss * 644 / 1e9)
                        if b.num_vss * 644 >= 2 * 126e6 else
                        "BVSS %.1f MB fits in L2: 512 MB L2 flush before every timed BFS" % (b.num_vss * 644 / 1e6)),
                    prep_s=prep["times"], parallelism=f"source-sharded x{world}" if world > 1 else "1 GPU")

    if args.partition == "rows" or args.virtual_ranks:
        run_partitioned(args, prep, B, L, lib, srcs_orig, perm, world, rank, local, workload, stream)
        return

    if args.impl == "reference":
        t0 = time.time()
        kind, cores, times, ctrs = cpu_reference_sample(prep, mine, lazy, budget_s=150.0, threads=threads,
                                                        max_steps=args.steps)
        # traversed edges per source (bookkeeping for the metric, outside the timed region)
        ev = [c["E"] for c in census_of(lib, L, b, prep, mine[: len(times)], lazy, args.pull)]
        hm = len(times) / sum(t / e for t, e in zip(times, ev)) / 1e9
        line = dict(metric="GTEPS (harmonic mean over sources)", value=round(hm, 6), unit="GTEPS",
                    n_gpus=1, steps=len(times), warmup=0, ms_per_step=round(1e3 * sum(times) / len(times), 3),
                    higher_is_better=True, scaling="weak", vs_baseline=None, dtype="u32", data="synthetic",
                    impl="reference", config=workload,
                    cpu_baseline=dict(value=round(hm, 6), unit="GTEPS", cores=cores, kind=kind,
                                      sample=f"{len(times)} of {args.steps} sources (bounded ~150 s), "
                                             f"R:src/bfs_engine.cpp run_{'lazy' if lazy else 'eager'} "
                                             f"workers={cores} num_warps={32 * cores}"),
                    e2e=dict(value=round(hm, 6), unit="GTEPS", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
        print(json.dumps(line), flush=True)
        return

    ecfg = L.EngineConfigT(L.MODE_LAZY if lazy else L.MODE_EAGER,
                           L.PULL_MMA if args.pull == "mma" else L.PULL_POPC, 0, 0, args.grid_ctas, args.threads)
    ctr = L.CountersT()
    # ---- census (untimed): deterministic counters + traversed edges per source ----
    census = census_of(lib, L, b, prep, mine, lazy, args.pull, args.threads, args.grid_ctas)
    if args.validate:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        off, tgt = prep["gp"].csr()
        csr = O.Csr(n, off, tgt)
        chk = mine[: args.validate]
        want, _ = O.reference_bfs_many(csr, chk)
        lv = np.zeros(n, np.uint32)
        for k, s in enumerate(chk):
            L.check(lib.blest_bfs(b.handle, int(s), C.byref(ecfg), lv.ctypes.data, C.byref(ctr), None, 0))
            assert np.array_equal(lv, want[k]), f"levels mismatch for source {int(s)}"
        log(f"validated {len(chk)} sources bit-exact against the CPU oracle")
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
    balg = np.array([b_alg(n, c["D"], c["P"], c["V"], c["L"], lazy) for c in census], np.float64)
    achieved = float(np.sum(balg) / total_s / 1e9)
    peak, peak_kind = load_peaks()
    value, elapsed = hm, total_s
    if world > 1:
        tt = torch.tensor([hm, total_s], dtype=torch.float64, device=coll_dev())
        allv = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(allv, tt)
        value = float(sum(x[0].item() for x in allv))
        elapsed = float(max(x[1].item() for x in allv))

    # ---- e2e through the C-ABI with host buffers (pinned) ----
    # blest_bfs_batch: the public many-sources call; source k's full level array is copied
    # to pinned host memory while source k+1 runs. Chunks of <= 16 sources (one pinned
    # buffer, reused; a 64-source / 4.3 GB buffer measured slower D2H: e2e 141 -> 74 GTEPS);
    # each source's time = its chunk's wall time / size.
    e2e = None
    if not args.no_e2e:
        chunk = max(1, min(16, len(mine), int(4e9 // (4 * max(n, 1)))))
        hl = torch.empty((chunk, n), dtype=torch.int32, pin_memory=True)
        hsrc = torch.empty(chunk, dtype=torch.int32, pin_memory=True)
        cbuf = (L.CountersT * chunk)()
        torch.cuda.synchronize()
        te = np.zeros(len(mine))
        for c0 in range(0, len(mine), chunk):
            part = np.ascontiguousarray(mine[c0:c0 + chunk], np.uint32)
            t0 = time.perf_counter()
            hsrc.numpy().view(np.uint32)[: len(part)] = part
            L.check(lib.blest_bfs_batch(b.handle, C.c_void_p(hsrc.data_ptr()), len(part), C.byref(ecfg),
                                        C.c_void_p(hl.data_ptr()), C.cast(cbuf, C.c_void_p)))
            te[c0:c0 + len(part)] = (time.perf_counter() - t0) / len(part)
        e2e_hm = len(te) / float(np.sum(te / E)) / 1e9
        e2e = dict(value=round(e2e_hm * world, 4), unit="GTEPS", h2d_bytes_per_step=4,
                   d2h_bytes_per_step=int(4 * n + 8 * 8 + 16),
                   note=f"blest_bfs_batch() in chunks of {chunk} sources: source ids in, every source's full "
                        "level array (pinned host) + counters out, host wall clock per chunk / chunk size")

    # ---- CPU baseline (rank 0, N = 1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        kind, cores, ctimes, _ = cpu_reference_sample(prep, mine, lazy, args.cpu_budget, threads, max_steps=8)
        chm = len(ctimes) / sum(tc / e for tc, e in zip(ctimes, E[: len(ctimes)])) / 1e9
        cpu = dict(value=round(chm, 6), unit="GTEPS", cores=cores, kind=kind,
                   sample=f"first {len(ctimes)} of the {len(mine)} timed sources (~{args.cpu_budget:.0f} s budget), "
                          f"run_{'lazy' if lazy else 'eager'} over the same BVSS arrays")

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
                          formula="648 D + 4 P + 4 n + 4 V + k (n/8) L (SURVEY 8(d))"),
            cpu_baseline=cpu, e2e=e2e, gpu_launches=int(launches),
            clocks=clk.summary(),
            detail=dict(grid=[g_ctas.value, g_thr.value], hm_gteps_rank0=round(hm, 4), mean_ms=round(1e3 * float(t.mean()), 4),
                        min_ms=round(1e3 * float(t.min()), 4), max_ms=round(1e3 * float(t.max()), 4),
                        mean_dequeues=int(np.mean([c["D"] for c in census])),
                        mean_levels=float(np.mean([c["L"] for c in census])),
                        mean_traversed_edges=int(E.mean()), arcs_per_s_G=round(2 * hm, 4)))
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_partitioned(args, prep, B, L, lib, srcs_orig, perm, world, rank, local, workload, stream):
    """Row-partitioned BFS: every rank owns a 32-aligned range of destination
    rows and its BVSS slice; per level a NCCL all-gather of the frontier diff words. Each
    step = one BFS from the next source over all ranks; value = harmonic-mean GTEPS of that
    distributed BFS (whole job), timed on each rank's device, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2512_21967_b200.multigpu import (GpuPartition, RowPartitionedBfs, nccl_allgather, partition_rows,
                                                 run_lockstep, words_per_rank)
    gp = prep["gp"]
    n = gp.num_vertices()
    deg = gp.out_degrees().astype(np.int64)
    srcs = perm.forward_map()[srcs_orig] if not perm.is_identity() else srcs_orig
    steps = srcs[args.warmup: args.warmup + args.steps]
    if args.virtual_ranks:
        G = args.virtual_ranks
        per = words_per_rank(n, G)
        parts = [GpuPartition(gp, lo, hi, per) for lo, hi in partition_rows(n, G)]
        run = lambda s: run_lockstep(parts, n, int(s))[0]
        mode = f"rows x{G} virtual ranks on 1 GPU"
    else:
        G = world
        lo, hi = partition_rows(n, G)[rank]
        part = GpuPartition(gp, lo, hi, words_per_rank(n, G))
        bfs = RowPartitionedBfs(part, n, nccl_allgather())
        run = lambda s: bfs.run(int(s))
        mode = f"rows x{G} ranks, {dist.get_backend().upper()} all-gather per level"
    del prep["b"]  # the single-GPU structure is not used by this mode
    for s in srcs[: args.warmup]:
        run(s)
    times, edges = [], []
    for s in steps:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = run(s)
        e1.record(stream)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        if args.virtual_ranks:
            reached = r != 0xFFFFFFFF
            e = int(deg[reached].sum()) // 2
        else:
            reached = r.levels != 0xFFFFFFFF
            e = int(deg[r.row_lo:r.row_hi][reached].sum())
        if world > 1 and not args.virtual_ranks:
            tt = torch.tensor([t, float(e)], dtype=torch.float64, device=coll_dev())
            tmax = tt.clone()
            dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
            t, e = float(tmax[0].item()), int(tt[1].item()) // 2
        times.append(t)
        edges.append(e)
    t = np.array(times)
    E = np.array(edges, np.float64)
    hm = len(t) / float(np.sum(t / E)) / 1e9
    if rank == 0:
        workload = dict(workload, parallelism=mode)
        print(json.dumps(dict(metric="GTEPS (harmonic mean over sources)", value=round(hm, 4), unit="GTEPS",
                              n_gpus=world, steps=len(t), warmup=args.warmup,
                              ms_per_step=round(1e3 * float(t.mean()), 4), higher_is_better=True,
                              scaling="strong", vs_baseline=None, dtype="u32", data="synthetic",
                              config=workload, detail=dict(mean_traversed_edges=int(E.mean())))), flush=True)


def census_of(lib, L, b, prep, sources, lazy, pull, threads=0, grid_ctas=0):
    """Per source: VSS dequeues D, pushes P, visited V, level iterations L and traversed
    undirected edges E (on the permuted graph, whose ids the level array uses)."""
    ecfg = L.EngineConfigT(L.MODE_LAZY if lazy else L.MODE_EAGER,
                           L.PULL_MMA if pull == "mma" else L.PULL_POPC, 0, 0, grid_ctas, threads)
    ctr = L.CountersT()
    lv_ptr = C.c_void_p()
    out = []
    for s in sources:
        L.check(lib.blest_bfs(b.handle, int(s), C.byref(ecfg), None, C.byref(ctr), None, 0))
        L.check(lib.blest_bfs_levels_device(b.handle, C.byref(lv_ptr)))
        e = prep["gp"].traversed_edges(lv_ptr.value)
        out.append(dict(D=ctr.vss_dequeues, P=ctr.queue_pushes, V=ctr.visited_count, L=ctr.trace_len, E=e))
    return out


if __name__ == "__main__":
    main()
