#!/bin/bash
mkdir -p gpurun_out
for x in $((1<<19)) $((1<<20)) $(((1<<20)+1024)); do
BLEST_XFLAGS=$x timeout 600 python tools/phase_profile.py --config c4 --sources 1 > gpurun_out/cl_e_$x.json 2> gpurun_out/cl_e_$x.err
python - $x <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/cl_e_{sys.argv[1]}.json"))
for r in d["runs"]:
    print(sys.argv[1], r["iterations"], r["total_us"], [(b["queue_lt"], b["mean_stage1_us"], b["mean_level_us"]) for b in r["queue_buckets"]])
PY
done
