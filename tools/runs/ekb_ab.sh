# eager batch size re-measured on C4 / C1 (alternating processes)
mkdir -p gpurun_out/ekb
for i in 1 2; do
  for c in c4 c1; do
    timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ekb/${c}_def_$i.json 2>/dev/null
    BLEST_LIB=variants/ekb2/libblest_b200.so timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/ekb/${c}_kb2_$i.json 2>/dev/null
    BLEST_LIB=variants/ekb8/libblest_b200.so timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/ekb/${c}_kb8_$i.json 2>/dev/null
  done
done
for f in gpurun_out/ekb/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], (d.get('parity') or {}).get('mismatches'))" 2>/dev/null); done
