# Round-2 evidence: tests, smoke, bench lines for every config, the reference arm, the
# multi-GPU rows mode (virtual ranks, torchrun gloo), timelines, ncu captures.
set -x
mkdir -p gpurun_out/final6
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final6/gputest.txt 2>&1; tail -2 gpurun_out/final6/gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6/smoke.txt 2>&1; tail -1 gpurun_out/final6/smoke.txt
timeout 900 python bench.py > gpurun_out/final6/bench_c2.json 2> gpurun_out/final6/bench_c2.err
timeout 900 python bench.py --impl reference --steps 8 --warmup 1 > gpurun_out/final6/ref_c2.json 2> gpurun_out/final6/ref_c2.err
timeout 600 python bench.py --config c1 --steps 16 > gpurun_out/final6/bench_c1.json 2> gpurun_out/final6/bench_c1.err
timeout 900 python bench.py --config c3 --steps 32 > gpurun_out/final6/bench_c3.json 2> gpurun_out/final6/bench_c3.err
timeout 1200 python bench.py --config c4 --steps 8 --cpu-budget 20 > gpurun_out/final6/bench_c4.json 2> gpurun_out/final6/bench_c4.err
timeout 2400 python bench.py --config c5 --steps 8 --warmup 2 --validate 8 > gpurun_out/final6/bench_c5.json 2> gpurun_out/final6/bench_c5.err
timeout 2400 python bench.py --config c5 --virtual-ranks 8 --steps 8 --warmup 2 --validate 8 > gpurun_out/final6/bench_c5_rows_v8.json 2> gpurun_out/final6/bench_c5_rows_v8.err
timeout 900 python bench.py --config c2 --virtual-ranks 8 --steps 16 --warmup 3 --validate 4 > gpurun_out/final6/bench_c2_rows_v8.json 2> gpurun_out/final6/bench_c2_rows_v8.err
timeout 900 python bench.py --config c3 --virtual-ranks 8 --steps 16 --warmup 3 --validate 4 > gpurun_out/final6/bench_c3_rows_v8.json 2> gpurun_out/final6/bench_c3_rows_v8.err
BLEST_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --config c2 --steps 8 --warmup 2 --validate 2 > gpurun_out/final6/bench_c2_n2_gloo.json 2> gpurun_out/final6/bench_c2_n2_gloo.err
timeout 900 python tools/rows_profile.py --config c5 --ranks 8 --sources 1 > gpurun_out/final6/rows_prof_c5_8.json 2> gpurun_out/final6/rows_prof_c5_8.err
timeout 600 python tools/phase_profile.py --config c2 --sources 2 > gpurun_out/final6/phase_c2.txt 2>&1
timeout 600 python tools/phase_profile.py --config c3 --mode lazy --sources 1 > gpurun_out/final6/phase_c3.txt 2>&1
timeout 1500 bash tools/profile.sh c2 > gpurun_out/final6/profile_c2.log 2>&1
timeout 1500 bash tools/profile.sh c3 > gpurun_out/final6/profile_c3.log 2>&1
ls -la gpurun_out/final6
