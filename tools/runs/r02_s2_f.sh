# rows engine first run: multigpu tests (fused virtual ranks, stepped, gloo world 2), lazy parity after the lazy_pull refactor
nvidia-smi --query-gpu=name,memory.used --format=csv
timeout 600 python -m pytest tests/test_gpu_multigpu.py -q -x --durations=10 > gpurun_out/gt_f_multi.txt 2>&1; echo multi rc=$?; tail -30 gpurun_out/gt_f_multi.txt
nvidia-smi --query-gpu=name,memory.used --format=csv
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_multigpu.py > gpurun_out/gt_f_all.txt 2>&1; echo all rc=$?; tail -5 gpurun_out/gt_f_all.txt
