timeout 1700 python -m pytest tests/test_gpu_io.py tests/test_gpu_scale.py -q -x --durations=15 > gpurun_out/gputest3.txt 2>&1; tail -25 gpurun_out/gputest3.txt
