# Round-end evidence: GPU tests, smoke, bench lines for every single-GPU config, the
# reference arm, ncu launch list + full capture of the C2 BFS kernel (profiles/).
bash tools/gpu_round.sh
mkdir -p gpurun_out/final
timeout 900 python bench.py > gpurun_out/final/bench_c2.json 2> gpurun_out/final/bench_c2.err
timeout 900 python bench.py --impl reference --steps 8 --warmup 1 > gpurun_out/final/ref_c2.json 2> gpurun_out/final/ref_c2.err
timeout 600 python bench.py --config c1 --steps 16 > gpurun_out/final/bench_c1.json 2> gpurun_out/final/bench_c1.err
timeout 900 python bench.py --config c3 --steps 32 > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err
timeout 900 python bench.py --config c4 --steps 8 --cpu-budget 20 > gpurun_out/final/bench_c4.json 2> gpurun_out/final/bench_c4.err
timeout 600 python tools/phase_profile.py --config c2 --sources 2 > gpurun_out/final/phase_c2.txt 2>&1
timeout 600 python tools/phase_profile.py --config c3 --sources 1 > gpurun_out/final/phase_c3.txt 2>&1
timeout 1200 bash tools/profile.sh c2 > gpurun_out/final/profile_c2.log 2>&1
timeout 1200 bash tools/profile.sh c3 > gpurun_out/final/profile_c3.log 2>&1
timeout 1800 python bench.py --config c5 --steps 4 --warmup 1 --no-cpu-baseline > gpurun_out/final/bench_c5.json 2> gpurun_out/final/bench_c5.err
