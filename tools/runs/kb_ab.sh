# lazy batch size and tail hand-out re-measured on the final kernel (alternating processes)
mkdir -p gpurun_out/kb
for i in 1 2; do
  for c in c2 c3; do
    timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/kb/${c}_def_$i.json 2>/dev/null
    BLEST_LIB=variants/kb4/libblest_b200.so timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/kb/${c}_kb4_$i.json 2>/dev/null
    BLEST_LIB=variants/kb2/libblest_b200.so timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/kb/${c}_kb2_$i.json 2>/dev/null
    BLEST_TAIL_DIV=4 timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/kb/${c}_td4_$i.json 2>/dev/null
    BLEST_TAIL_DIV=16 timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/kb/${c}_td16_$i.json 2>/dev/null
  done
done
for f in gpurun_out/kb/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], (d.get('parity') or {}).get('mismatches'))" 2>/dev/null); done
