"""CPU checks of bench.py's bookkeeping (no GPU): the algorithmic-bytes formula of SURVEY
§8(d), the config table, and the clock sampler's timed-window filter."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_b_alg_formula():
    # 648 D + 4 P + 4 n + 4 V + k (n/8) L, k = 2 lazy / 1 eager
    n, D, P, V, L = 1 << 20, 1000, 50, 900, 7
    assert bench.b_alg(n, D, P, V, L, True) == 648 * D + 4 * P + 4 * n + 4 * V + 2 * (n // 8) * L
    assert bench.b_alg(n, D, P, V, L, False) == 648 * D + 4 * P + 4 * n + 4 * V + (n // 8) * L


def test_configs_cover_baseline():
    assert set(bench.CONFIGS) == {"c1", "c2", "c3", "c4", "c5"}
    kind, prm, ordering, _ = bench.CONFIGS["c2"]
    assert kind == "rmat" and prm["scale"] == 24 and prm["ef"] == 16 and ordering == "auto"
    assert bench.CONFIGS["c5"][1]["scale"] == 27
    assert bench.CONFIGS["c4"][1]["rows"] * bench.CONFIGS["c4"][1]["cols"] == 4096 * 8192


def test_clock_sampler_window():
    c = bench.ClockSampler(0)
    row = lambda mhz, thr="Not Active": [str(mhz), "1965", "Not Active", thr, "Not Active", "Not Active"]
    c.rows = [(1.0, row(1000)), (2.0, row(1965)), (2.5, row(1900, "Active")), (9.0, row(500))]
    c.t0, c.t1 = 1.9, 2.6
    s = c.summary()
    assert s["samples"] == 2 and s["sm_mhz"] == (1965 + 1900) / 2
    assert s["reasons"] == ["hw_thermal_slowdown"]
    c.t0, c.t1 = 5.0, 5.01  # shorter than the sampling period: nearest samples
    assert c.summary()["samples"] == 3
