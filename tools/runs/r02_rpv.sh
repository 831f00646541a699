#!/bin/bash
# stage 2: vectorised real_ptrs loads; A/B against the HEAD build (separate processes, alternating)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "phase_variants or dense_levels or c1_rmat16" > gpurun_out/rp_par.txt 2>&1; echo "par rc=$?"; tail -2 gpurun_out/rp_par.txt
for r in 1 2; do
for lib in variants/base/libblest_b200.so paper_2512_21967_b200/libblest_b200.so; do
for c in c2 c3; do
BLEST_LIB=$lib timeout 900 python bench.py --config $c --steps 32 --warmup 3 --no-cpu-baseline --no-e2e --validate 2 > gpurun_out/rp_$c.json 2> gpurun_out/rp_$c.err
python -c "import json;d=json.load(open('gpurun_out/rp_$c.json'));print('$c', '$lib', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity']['mismatches'])" || tail -3 gpurun_out/rp_$c.err
done
done
done
