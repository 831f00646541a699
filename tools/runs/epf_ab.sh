# eager sparse-level push-time L2 prefetch on/off with kBatch 2
mkdir -p gpurun_out/epf
for i in 1 2; do
  for c in c4 c1; do
    timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/epf/${c}_on_$i.json 2>/dev/null
    BLEST_XFLAGS=1024 timeout 900 python bench.py --config $c --steps 8 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/epf/${c}_off_$i.json 2>/dev/null
  done
done
for f in gpurun_out/epf/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])" 2>/dev/null); done
