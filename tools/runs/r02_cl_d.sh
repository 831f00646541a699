#!/bin/bash
# grid eager barrier study on C4: probes around the grid barrier, prefetch on/off
mkdir -p gpurun_out
for x in 131072 262144 $((131072+1024)) $((262144+1024)) $((65536+1024)); do
BLEST_XFLAGS=$x timeout 600 python tools/phase_profile.py --config c4 --sources 1 > gpurun_out/cl_d_$x.json 2> gpurun_out/cl_d_$x.err
python - $x <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/cl_d_{sys.argv[1]}.json"))
for r in d["runs"]:
    print(sys.argv[1], r["iterations"], r["total_us"], [(b["queue_lt"], b["mean_stage1_us"], b["mean_level_us"]) for b in r["queue_buckets"]])
PY
done
