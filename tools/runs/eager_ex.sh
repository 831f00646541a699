# eager exhaustion exit: parity, then C4 / C1 (eager by default) A/B against the previous build, C3 with the eager engine
mkdir -p gpurun_out/ee
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/ee/test.txt 2>&1; tail -2 gpurun_out/ee/test.txt
for i in 1 2; do
  BLEST_LIB=variants/base2/libblest_b200.so timeout 900 python bench.py --config c4 --steps 8 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ee/c4_base_$i.json 2> gpurun_out/ee/c4_base_$i.err
  timeout 900 python bench.py --config c4 --steps 8 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ee/c4_new_$i.json 2> gpurun_out/ee/c4_new_$i.err
  BLEST_LIB=variants/base2/libblest_b200.so timeout 600 python bench.py --config c1 --steps 16 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ee/c1_base_$i.json 2> gpurun_out/ee/c1_base_$i.err
  timeout 600 python bench.py --config c1 --steps 16 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ee/c1_new_$i.json 2> gpurun_out/ee/c1_new_$i.err
done
timeout 900 python bench.py --config c3 --mode eager --steps 16 --warmup 3 --validate 4 --no-cpu-baseline --no-e2e > gpurun_out/ee/c3e_new.json 2> gpurun_out/ee/c3e_new.err
BLEST_EXHAUST=0 timeout 900 python bench.py --config c3 --mode eager --steps 16 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ee/c3e_off.json 2> gpurun_out/ee/c3e_off.err
for f in gpurun_out/ee/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['detail'].get('mean_unpulled'), (d.get('parity') or {}).get('mismatches'))"); done
for i in 1 2; do
  BLEST_LIB=variants/base2/libblest_b200.so timeout 600 python bench.py --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ee/c2_base_$i.json 2> /dev/null
  timeout 600 python bench.py --steps 32 --warmup 3 --validate 0 --no-cpu-baseline --no-e2e > gpurun_out/ee/c2_new_$i.json 2> /dev/null
done
for f in gpurun_out/ee/c2_*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"); done
