SKIP_TESTS=1 bash tools/gpu_round.sh
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 900 $B --config c4 --steps 4 > gpurun_out/c4_t512.json 2>/dev/null
timeout 900 $B --config c4 --steps 4 --threads 1024 > gpurun_out/c4_t1024.json 2>/dev/null
timeout 900 $B --config c4 --steps 4 --threads 256 > gpurun_out/c4_t256.json 2>/dev/null
timeout 900 $B --config c4 --steps 4 --grid-ctas 74 > gpurun_out/c4_g74.json 2>/dev/null
