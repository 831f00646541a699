bash tools/gpu_round.sh
mkdir -p gpurun_out/final
timeout 900 python bench.py > gpurun_out/final/bench_c2b.json 2> gpurun_out/final/bench_c2b.err
timeout 600 python bench.py --config c1 --steps 16 > gpurun_out/final/bench_c1b.json 2> gpurun_out/final/bench_c1b.err
