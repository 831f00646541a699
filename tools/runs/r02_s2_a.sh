# session 2 first GPU check: full -m gpu suite, C2 bench (default validate), reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/gputest_s2.txt 2>&1; echo pytest rc=$?; tail -30 gpurun_out/gputest_s2.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; echo bench rc=$?; tail -5 gpurun_out/b_c2.err; cat gpurun_out/b_c2.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; echo ref rc=$?; tail -3 gpurun_out/ref_c2.err; cat gpurun_out/ref_c2.json
