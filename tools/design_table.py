"""Print DESIGN.md §5's end-state table from a set of committed bench lines.

    python tools/design_table.py r02_final6        # reads profiles/r02_final6_*.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def line(tag, name):
    with open(os.path.join(ROOT, "profiles", f"{tag}_{name}.json")) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def row(label, engine, d, frac=None, cpu="—", bold=False):
    pr = d["parity"]
    fr = frac if frac is not None else (f"{d['roofline']['frac']:.3f}" if d.get("roofline") else "—")
    val = f"{d['value']:.1f}" if d["value"] >= 10 else f"{d['value']:.3f}"
    e2e = d["e2e"]["value"]
    e2e = f"{e2e:.1f}" if e2e >= 10 else f"{e2e:.3f}"
    if bold:
        val, fr = f"**{val}**", f"**{fr}**"
    return (f"| {label} | {engine} | {d['ms_per_step']:.3f} | {val} | {fr} | {e2e} | "
            f"{pr['checked']} / {pr['checked']} | {cpu} |")


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02_final6"
    c1, c2, c3, c4, c5 = (line(tag, f"bench_c{i}") for i in range(1, 6))
    ref = line(tag, "reference_c2")
    out = ["| config | engine | ms / BFS | GTEPS (HM) | roofline frac | e2e GTEPS | parity | CPU baseline |",
           "|---|---|---|---|---|---|---|---|",
           row("C2 Kron-24 (headline, 64 sources)", "lazy", c2,
               cpu=f"{c2['cpu_baseline']['value']:.3f} (reference `run_lazy`, 16 threads)", bold=True),
           row("C1 RMAT-16 (L2 flushed per BFS)", "eager", c1, cpu=f"{c1['cpu_baseline']['value']:.3f}"),
           row("C3 urand-24 (RCM)", "lazy (+ exhaustion exit)", c3,
               frac=f"{c3['roofline']['frac']:.3f} (pulled VSSs only)", cpu=f"{c3['cpu_baseline']['value']:.3f}"),
           row("C4 grid 4096×8192 (RCM, ~8.6 K levels)", "eager", c4, cpu=f"{c4['cpu_baseline']['value']:.4f}"),
           row("C5 Kron-27 on one GPU (28 GB BVSS, 43.7 M VSS)", "lazy", c5,
               cpu=f"{c5['cpu_baseline']['value']:.3f} (`reference_bfs`, 1 core: the reference engine is "
                   "invalid at ≥ 2^25 VSSs)")]
    for name, label, eng in (("bench_c5_rows_v8", "C5, rows mode, 8 virtual ranks on one GPU", "rows"),
                             ("bench_c3_rows_v8", "C3, rows mode, 8 virtual ranks on one GPU", "rows (+ exit)"),
                             ("bench_c2_rows_v8", "C2, rows mode, 8 virtual ranks on one GPU", "rows")):
        out.append(row(label, eng, line(tag, name), frac="—"))
    out.append(f"| reference arm C2 (`--impl reference`, host only) | reference `run_lazy` | "
               f"{ref['ms_per_step']:.0f} | {ref['value']:.3f} | — | — | engine vs `reference_bfs` | — |")
    print("\n".join(out))


if __name__ == "__main__":
    main()
