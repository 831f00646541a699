#!/bin/bash
# C4 (grid, RCM, eager): per-level time bucketed by queue size
mkdir -p gpurun_out
BLEST_XFLAGS=64 timeout 600 python tools/phase_profile.py --config c4 --sources 1 > gpurun_out/c4_hist.json 2> gpurun_out/c4_hist.err; echo rc=$?
python - <<'PY'
import json
d = json.load(open("gpurun_out/c4_hist.json"))
for r in d["runs"]:
    print(r["source"], r["iterations"], r["total_us"])
    for b in r["queue_buckets"]:
        print(b)
PY
