# eager threads per CTA (occupancy) with kBatch 2, C4 / C1
mkdir -p gpurun_out/eth
for i in 1 2; do
  for c in c4 c1; do
    for t in 512 1024 256; do
      timeout 900 python bench.py --config $c --threads $t --steps 8 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/eth/${c}_t${t}_$i.json 2>/dev/null
    done
  done
done
timeout 900 python bench.py --config c3 --mode eager --steps 16 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/eth/c3e_t512.json 2>/dev/null
timeout 900 python bench.py --config c3 --mode eager --threads 1024 --steps 16 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/eth/c3e_t1024.json 2>/dev/null
for f in gpurun_out/eth/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], (d.get('parity') or {}).get('mismatches'), d['detail'].get('grid'))" 2>/dev/null); done
