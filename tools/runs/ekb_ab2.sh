# eager batch size 1/2/3 vs 4 on C4 / C1 / C3 (eager engine)
mkdir -p gpurun_out/ekb2
for i in 1 2; do
  for c in c4 c1; do
    timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ekb2/${c}_def_$i.json 2>/dev/null
    for v in 1 2 3; do
      BLEST_LIB=variants/ekb$v/libblest_b200.so timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/ekb2/${c}_kb${v}_$i.json 2>/dev/null
    done
  done
done
timeout 900 python bench.py --config c3 --mode eager --steps 16 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ekb2/c3e_def.json 2>/dev/null
for v in 1 2 3; do
  BLEST_LIB=variants/ekb$v/libblest_b200.so timeout 900 python bench.py --config c3 --mode eager --steps 16 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/ekb2/c3e_kb$v.json 2>/dev/null
done
for f in gpurun_out/ekb2/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], (d.get('parity') or {}).get('mismatches'))" 2>/dev/null); done
