bash tools/gpu_round.sh
mkdir -p gpurun_out/final
timeout 900 python bench.py --config c3 --steps 32 > gpurun_out/final/bench_c3_b200.json 2> gpurun_out/final/bench_c3_b200.err
timeout 600 python tools/phase_profile.py --config c3 --mode lazy --sources 1 > gpurun_out/final/phase_c3_lazy.txt 2>&1
timeout 1200 bash tools/profile.sh c3 > gpurun_out/final/profile_c3.log 2>&1
timeout 600 python bench.py --steps 16 --no-cpu-baseline > gpurun_out/final/bench_c2_check.json 2>/dev/null
