bash tools/gpu_round.sh
B="python bench.py --no-cpu-baseline --no-e2e --steps 16"
timeout 600 $B > gpurun_out/h2_c2.json 2>gpurun_out/h2_c2.err
BLEST_SIGMA=0 timeout 600 $B > gpurun_out/h2_c2_nosig.json 2>/dev/null
BLEST_HOT=524288 timeout 600 $B > gpurun_out/h2_c2_hot512k.json 2>/dev/null
BLEST_HOT=2097152 timeout 600 $B > gpurun_out/h2_c2_hot2m.json 2>/dev/null
timeout 600 python tools/phase_profile.py --config c2 --sources 2 > gpurun_out/h2_phase.txt 2>&1
