# cp.async-staged dense pull (variants/astage) vs default: parity subset, then alternating C2/C3 benches
mkdir -p gpurun_out/as
BLEST_LIB=variants/astage/libblest_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "lazy or engine or variants" > gpurun_out/as/test.txt 2>&1; tail -2 gpurun_out/as/test.txt
for i in 1 2; do
  for c in c2 c3; do
    timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/as/${c}_def_$i.json 2> gpurun_out/as/${c}_def_$i.err
    BLEST_LIB=variants/astage/libblest_b200.so timeout 600 python bench.py --config $c --steps 32 --warmup 3 --validate 4 --no-cpu-baseline --no-e2e > gpurun_out/as/${c}_as_$i.json 2> gpurun_out/as/${c}_as_$i.err
  done
done
BLEST_LIB=variants/astage/libblest_b200.so timeout 600 python tools/phase_profile.py --config c2 --mode lazy --sources 1 > gpurun_out/as/phase_c2_as.txt 2>&1
for f in gpurun_out/as/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], (d.get('parity') or {}).get('mismatches'))"); done
