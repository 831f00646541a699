# rows-engine exhaustion exit: multi-GPU tests, then rows-mode benches (8 virtual ranks)
mkdir -p gpurun_out/rx
timeout 1200 python -m pytest tests/test_gpu_multigpu.py -q -m gpu -x > gpurun_out/rx/test.txt 2>&1; tail -3 gpurun_out/rx/test.txt
timeout 900 python bench.py --config c3 --virtual-ranks 8 --steps 16 --warmup 3 --validate 4 > gpurun_out/rx/c3_rows_v8.json 2> gpurun_out/rx/c3_rows_v8.err
BLEST_EXHAUST=0 timeout 900 python bench.py --config c3 --virtual-ranks 8 --steps 16 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/rx/c3_rows_v8_off.json 2> gpurun_out/rx/c3_rows_v8_off.err
timeout 900 python bench.py --config c2 --virtual-ranks 8 --steps 16 --warmup 3 --validate 4 > gpurun_out/rx/c2_rows_v8.json 2> gpurun_out/rx/c2_rows_v8.err
for f in gpurun_out/rx/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), (d.get('parity') or {}).get('mismatches'), (d.get('e2e') or {}).get('value'))"); done
