#!/bin/bash
# eager warp-local queues: parity, then C4 / C1 against the HEAD build (separate processes, alternating)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cpp_facade.py -m gpu -x -q > gpurun_out/wl_par.txt 2>&1; echo "par rc=$?"; tail -2 gpurun_out/wl_par.txt
for r in 1 2; do
for lib in variants/base/libblest_b200.so paper_2512_21967_b200/libblest_b200.so; do
BLEST_LIB=$lib timeout 900 python bench.py --config c4 --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --validate 2 > gpurun_out/wl_c4.json 2> gpurun_out/wl_c4.err
python -c "import json;d=json.load(open('gpurun_out/wl_c4.json'));print('c4', '$lib', d['value'], d['ms_per_step'], d['parity']['mismatches'])" || tail -3 gpurun_out/wl_c4.err
BLEST_LIB=$lib timeout 900 python bench.py --config c1 --steps 32 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/wl_c1.json 2> gpurun_out/wl_c1.err
python -c "import json;d=json.load(open('gpurun_out/wl_c1.json'));print('c1', '$lib', d['value'], d['ms_per_step'], d['parity']['mismatches'])" || tail -3 gpurun_out/wl_c1.err
done
done
BLEST_XFLAGS=64 timeout 600 python tools/phase_profile.py --config c4 --sources 1 > gpurun_out/wl_hist.json 2> gpurun_out/wl_hist.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/wl_hist.json"))
for r in d["runs"]:
    print(r["iterations"], r["total_us"], [(b["queue_lt"], b["mean_stage1_us"], b["mean_level_us"]) for b in r["queue_buckets"]])
PY
