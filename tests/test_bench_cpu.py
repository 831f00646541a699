"""CPU checks of bench.py's bookkeeping (no GPU): the algorithmic-bytes formula of SURVEY
§8(d), the config table, and the clock sampler's timed-window filter."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_b_alg_formula():
    # 648 D + 4 P + 4 n + 4 V + k (n/8) L, k = 2 lazy (V_curr + V_next sweep); eager never
    # sweeps Θ(n) per level on the B200 (triple-buffered frontier), so k = 0
    n, D, P, V, L = 1 << 20, 1000, 50, 900, 7
    assert bench.b_alg(n, D, P, V, L, True) == 648 * D + 4 * P + 4 * n + 4 * V + 2 * (n // 8) * L
    assert bench.b_alg(n, D, P, V, L, False) == 648 * D + 4 * P + 4 * n + 4 * V


def test_batch_d2h_bytes_follows_the_width_rule():
    """blest_bfs_batch's narrow transfers (BfsEngine::run_batch): 1 byte per vertex (+ the
    8-byte deepest level) while levels fit; a source past 254 levels is re-copied as u32 once
    its copy lands (two sources later) and widens the sources launched after that."""
    n = 1000
    assert bench.batch_d2h_bytes([7] * 5, n, packed=False) == 4 * n * 5
    assert bench.batch_d2h_bytes([7] * 5, n, packed=True) == 5 * (n + 8)
    # 4 deep sources: 0, 1 go at 1 byte (+ u32 re-copy each); 2, 3 at 2 bytes
    assert bench.batch_d2h_bytes([300] * 4, n, True) == 2 * (n + 8 + 4 * n) + 2 * (2 * n + 8)
    # past 65 534 levels: u32 from then on
    assert bench.batch_d2h_bytes([70000] * 4, n, True) == 2 * (n + 8 + 4 * n) + 2 * 4 * n


def test_configs_cover_baseline():
    assert set(bench.CONFIGS) == {"c1", "c2", "c3", "c4", "c5"}
    kind, prm, ordering, _ = bench.CONFIGS["c2"]
    assert kind == "rmat" and prm["scale"] == 24 and prm["ef"] == 16 and ordering == "auto"
    assert bench.CONFIGS["c5"][1]["scale"] == 27
    assert bench.CONFIGS["c4"][1]["rows"] * bench.CONFIGS["c4"][1]["cols"] == 4096 * 8192


def test_clock_sampler_window():
    c = bench.ClockSampler(0)
    thermal = dict(bench.ClockSampler.REASONS)["hw_thermal_slowdown"]
    c.rows = [(1.0, [1000, 1965, 0]), (2.0, [1965, 1965, 0]), (2.5, [1900, 1965, thermal]), (9.0, [500, 1965, 0])]
    c.t0, c.t1 = 1.9, 2.6
    s = c.summary()
    assert s["samples"] == 2 and s["sm_mhz"] == (1965 + 1900) / 2
    assert s["reasons"] == ["hw_thermal_slowdown"]
    c.t0, c.t1 = 5.0, 5.01  # shorter than the sampling period: nearest samples
    assert c.summary()["samples"] == 3
    assert bench.ClockSampler(0).summary()["reasons"] == ["unsampled"]


def test_reference_arm_cpu_only(tmp_path):
    """--impl reference runs on the host alone: the product library is never loaded, the
    structure comes from the CPU oracle, and the reference engine's levels are checked."""
    import json
    import subprocess
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '3',"
            " '--warmup', '1']; runpy.run_path('bench.py', run_name='__main__');"
            " maps = open('/proc/self/maps').read();"
            " assert 'libblest_b200' not in maps, 'product library mapped'; assert 'libblest_ref' in maps")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 3 and line["warmup"] == 1
    assert line["parity"]["mismatches"] == 0 and line["value"] > 0
    assert line["config"]["workload"] == "c1" and line["cpu_baseline"]["kind"] == "reference"
