# lazy CTA size: 2 x 512 (default) vs 1 x 1024 threads per SM
mkdir -p gpurun_out/lth
for i in 1 2; do
  for c in c2 c3; do
    timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/lth/${c}_t512_$i.json 2>/dev/null
    timeout 600 python bench.py --config $c --threads 1024 --steps 32 --warmup 3 --validate 2 --no-cpu-baseline --no-e2e > gpurun_out/lth/${c}_t1024_$i.json 2>/dev/null
  done
done
for f in gpurun_out/lth/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], (d.get('parity') or {}).get('mismatches'), d['detail'].get('grid'))" 2>/dev/null); done
