"""Summarise gpurun_out/ ncu outputs into profiles/ (tracked): the launch list (per kernel
name: launches, total and share of device time) and the full capture's key metrics
(duration, DRAM bytes read/write, throughputs, occupancy, L1/L2 hit rates, stall reasons).

    python tools/summarize_profile.py c2 r01
"""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").strip()
        ns = float(d["Metric Value"].replace(",", ""))
        if d.get("Metric Unit") == "us":
            ns *= 1e3
        elif d.get("Metric Unit") == "ms":
            ns *= 1e6
        e = out.setdefault(name, {"launches": 0, "total_ns": 0.0})
        e["launches"] += 1
        e["total_ns"] += ns
    tot = sum(e["total_ns"] for e in out.values()) or 1.0
    for e in out.values():
        e["share"] = round(e["total_ns"] / tot, 4)
        e["mean_us"] = round(e["total_ns"] / e["launches"] / 1e3, 2)
    return dict(sorted(out.items(), key=lambda kv: -kv[1]["total_ns"]))


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))

    def num(k, scale_to=None):
        if k not in d or d[k] in ("", "n/a"):
            return None
        v = float(d[k].replace(",", ""))
        unit = u.get(k, "")
        mult = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1e-6, "msecond": 1e-3,
                "nsecond": 1e-9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}.get(unit, 1)
        return v * mult

    keys = {
        "duration_s": "gpu__time_duration.sum",
        "dram_bytes_read": "dram__bytes_read.sum",
        "dram_bytes_write": "dram__bytes_write.sum",
        "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1_hit_rate_pct": "l1tex__t_sector_hit_rate.pct",
        "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "registers_per_thread": "launch__registers_per_thread",
        "grid_size": "launch__grid_size",
        "block_size": "launch__block_size",
        "red_instructions": "smsp__inst_executed_op_global_red.sum",
        "lts_sectors_op_red": "lts__t_sectors_op_red.sum",
        "lts_sectors_op_atom": "lts__t_sectors_op_atom.sum",
        "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "imma_pipe_inst": "sm__inst_executed_pipe_tensor_op_imma.sum",
    }
    out = {k: num(v) for k, v in keys.items()}
    out["kernel"] = re.sub(r"\(.*", "", vals[hdr.index("Kernel Name")]) if "Kernel Name" in hdr else None
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k]) for k in hdr
          if re.match(r"smsp__pcsamp_warps_issue_stalled_[a-z_]+$", k) and not k.endswith("not_issued")
          and d[k] not in ("", "n/a")}
    tot = sum(st.values()) or 1.0
    out["stall_share"] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:8]}
    if out["dram_bytes_read"] is not None:
        out["dram_bytes_total"] = out["dram_bytes_read"] + (out["dram_bytes_write"] or 0)
    return out


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    res = {"config": cfg}
    lp = os.path.join(ROOT, "gpurun_out", f"launches_{cfg}.csv")
    if os.path.exists(lp):
        res["launch_list"] = launches(lp)
    fp = os.path.join(ROOT, "gpurun_out", f"full_{cfg}.ncu-rep")
    if os.path.exists(fp):
        res["full_capture"] = fc = full(fp)
        k = fc.get("kernel") or ""
        if "k_bfs_" in k and fc.get("dram_bytes_total"):
            # bench.py's roofline.traffic: DRAM bytes of one BFS launch (read + write)
            engine = "lazy" if "lazy" in k else "eager"
            full_name = subprocess.run(["ncu", "-i", fp, "--page", "raw", "--csv"], capture_output=True,
                                       text=True).stdout
            pull = "mma" if "<1," in full_name or "(int)1," in full_name else "popc"
            with open(os.path.join(ROOT, "profiles", f"traffic_{cfg}.json"), "w") as f:
                json.dump(dict(config=cfg, engine=engine, pull=pull, kernel=k,
                               dram_bytes_per_launch=int(fc["dram_bytes_total"]),
                               source=f"ncu --set full capture gpurun_out/full_{cfg}.ncu-rep ({tag})"), f, indent=1)
    with open(os.path.join(ROOT, "profiles", f"{tag}_{cfg}_ncu_summary.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
