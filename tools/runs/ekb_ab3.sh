# per-level-kind eager batch (dense 3 / sparse 1) vs uniform 1 and the previous 4
mkdir -p gpurun_out/ekb3
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/ekb3/test.txt 2>&1; tail -2 gpurun_out/ekb3/test.txt
for i in 1 2; do
  for c in c4 c1; do
    timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/ekb3/${c}_new_$i.json 2>/dev/null
    BLEST_LIB=variants/ekb1/libblest_b200.so timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ekb3/${c}_kb1_$i.json 2>/dev/null
    BLEST_LIB=variants/base2/libblest_b200.so timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ekb3/${c}_kb4_$i.json 2>/dev/null
  done
  timeout 900 python bench.py --config c3 --mode eager --steps 16 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/ekb3/c3e_new_$i.json 2>/dev/null
  BLEST_LIB=variants/ekb3/libblest_b200.so timeout 900 python bench.py --config c3 --mode eager --steps 16 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ekb3/c3e_kb3_$i.json 2>/dev/null
done
for f in gpurun_out/ekb3/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], (d.get('parity') or {}).get('mismatches'))" 2>/dev/null); done
