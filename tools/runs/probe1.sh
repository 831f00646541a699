mkdir -p gpurun_out/p1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "exhaustion or narrow" > gpurun_out/p1/test.txt 2>&1; tail -2 gpurun_out/p1/test.txt
timeout 600 python tools/phase_profile.py --config c3 --mode lazy --sources 2 > gpurun_out/p1/phase_c3_lazy.txt 2>&1
