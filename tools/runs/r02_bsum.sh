#!/bin/bash
# grid_barrier_sum (BLEST_XFLAGS bit 21): parity under the switch, then same-process A/B
mkdir -p gpurun_out
BLEST_XFLAGS=2097152 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/bs_par.txt 2>&1; echo "par rc=$?"; tail -2 gpurun_out/bs_par.txt
for c in c4 c1 c2; do
timeout 900 python tools/ab.py --config $c --sources 6 --rounds 3 --variants '{"cg": {}, "sum": {"BLEST_XFLAGS": "2097152"}}' > gpurun_out/bs_ab_$c.json 2> gpurun_out/bs_ab_$c.err
python - $c <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bs_ab_{sys.argv[1]}.json"))
for k, v in d["variants"].items():
    print(sys.argv[1], k, v["ms_mean"], v["gteps_hm"], v["ms_round_means"])
PY
done
