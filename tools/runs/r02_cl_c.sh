#!/bin/bash
# grid eager chain study on C4: tstamp slot 1 = CTA 0 warp 0 after each phase
mkdir -p gpurun_out
for c in 0 1; do
for x in 4096 8192 16384 32768 65536; do
BLEST_CLUSTER=$c BLEST_XFLAGS=$x timeout 600 python tools/phase_profile.py --config c4 --sources 1 > gpurun_out/cl_c_$x.json 2> gpurun_out/cl_c_$x.err
python - $x $c <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/cl_c_{sys.argv[1]}.json"))
for r in d["runs"]:
    print(sys.argv[2], sys.argv[1], r["iterations"], r["total_us"], [(b["queue_lt"], b["mean_stage1_us"], b["mean_level_us"]) for b in r["queue_buckets"]])
PY
done
done
