# round-2 check: GPU tests (incl. scale), C2 bench with parity, tail A/B, reference arm
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest2.txt 2>&1; tail -3 gpurun_out/gputest2.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; tail -2 gpurun_out/b_c2.err
for t in 0 8 0 8; do BLEST_TAIL_DIV=$t timeout 600 python bench.py --steps 20 --warmup 5 --validate 0 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tail', $t, d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"; done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; tail -2 gpurun_out/ref_c2.err
