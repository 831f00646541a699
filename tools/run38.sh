SKIP_TESTS=1 bash tools/gpu_round.sh
B="python bench.py --no-cpu-baseline --no-e2e --steps 16"
timeout 600 $B > gpurun_out/sw_base.json 2>/dev/null
BLEST_HOT=262144 timeout 600 $B > gpurun_out/sw_hot256k.json 2>/dev/null
BLEST_HOT=4194304 timeout 600 $B > gpurun_out/sw_hot4m.json 2>/dev/null
BLEST_LIB=build/exp/m3/libblest_b200.so timeout 600 $B > gpurun_out/sw_m3.json 2>/dev/null
timeout 600 $B --threads 256 > gpurun_out/sw_t256.json 2>/dev/null
