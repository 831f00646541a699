# lazy exhaustion exit: parity (engine tests), then C3 / C2 A/B: base build (HEAD~), new build, new with BLEST_EXHAUST=0
mkdir -p gpurun_out/ex
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -m gpu -x > gpurun_out/ex/test.txt 2>&1; tail -2 gpurun_out/ex/test.txt
for i in 1 2; do
  for c in c3 c2; do
    BLEST_LIB=variants/base/libblest_b200.so timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ex/${c}_base_$i.json 2> gpurun_out/ex/${c}_base_$i.err
    timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ex/${c}_new_$i.json 2> gpurun_out/ex/${c}_new_$i.err
    BLEST_EXHAUST=0 timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ex/${c}_off_$i.json 2> gpurun_out/ex/${c}_off_$i.err
  done
done
timeout 600 python bench.py --config c3 --steps 32 --warmup 3 > gpurun_out/ex/c3_full.json 2> gpurun_out/ex/c3_full.err
for f in gpurun_out/ex/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['detail'].get('mean_unpulled'), (d.get('parity') or {}).get('mismatches'))"); done
