#!/bin/bash
# rows kernel stage 2b: vectorised real_ptrs loads; parity + A/B on C2 with 8 virtual ranks
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/rr_par.txt 2>&1; echo "par rc=$?"; tail -2 gpurun_out/rr_par.txt
for r in 1 2; do
for lib in variants/base/libblest_b200.so paper_2512_21967_b200/libblest_b200.so; do
BLEST_LIB=$lib timeout 900 python bench.py --config c2 --virtual-ranks 8 --steps 16 --warmup 3 --no-cpu-baseline --no-e2e --validate 2 > gpurun_out/rr.json 2> gpurun_out/rr.err
python -c "import json;d=json.load(open('gpurun_out/rr.json'));print('c2 v8', '$lib', d['value'], d['ms_per_step'], d['parity']['mismatches'])" || tail -3 gpurun_out/rr.err
done
done
