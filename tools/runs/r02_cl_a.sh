#!/bin/bash
# cluster engine (bfs_cluster.cu): parity with BLEST_CLUSTER=1, then C4/C1 timings both ways
mkdir -p gpurun_out
BLEST_CLUSTER=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/cl_a_par.txt 2>&1; echo "par rc=$?"; tail -3 gpurun_out/cl_a_par.txt
BLEST_CLUSTER=1 BLEST_XFLAGS=64 timeout 600 python tools/phase_profile.py --config c4 --sources 1 > gpurun_out/cl_a_c4_hist.json 2> gpurun_out/cl_a_c4_hist.err; echo rc=$?; tail -3 gpurun_out/cl_a_c4_hist.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/cl_a_c4_hist.json"))
for r in d["runs"]:
    print(r["source"], r["iterations"], r["total_us"])
    for b in r["queue_buckets"]:
        print(b)
PY
for c in 1 0; do
BLEST_CLUSTER=$c timeout 900 python bench.py --config c4 --steps 4 --warmup 3 --no-cpu-baseline --validate 2 > gpurun_out/cl_a_c4_$c.json 2> gpurun_out/cl_a_c4_$c.err
python -c "import json;d=json.load(open('gpurun_out/cl_a_c4_$c.json'));print('c4 cluster=$c', d['value'], d['ms_per_step'], d.get('parity'))"
BLEST_CLUSTER=$c timeout 900 python bench.py --config c1 --steps 16 --warmup 3 --no-cpu-baseline > gpurun_out/cl_a_c1_$c.json 2> gpurun_out/cl_a_c1_$c.err
python -c "import json;d=json.load(open('gpurun_out/cl_a_c1_$c.json'));print('c1 cluster=$c', d['value'], d['ms_per_step'], d.get('parity'))"
done
