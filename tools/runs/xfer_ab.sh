# narrow level transfers: parity tests, then e2e A/B (BLEST_D2H_PACK=1 vs 0) on C2 and C5
mkdir -p gpurun_out/xf
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "batch" > gpurun_out/xf/test.txt 2>&1; tail -2 gpurun_out/xf/test.txt
for i in 1 2; do for p in 1 0; do
  BLEST_D2H_PACK=$p timeout 600 python bench.py --steps 32 --warmup 3 --validate 0 --no-cpu-baseline > gpurun_out/xf/c2_p${p}_$i.json 2> gpurun_out/xf/c2_p${p}_$i.err
done; done
for p in 1 0; do
  BLEST_D2H_PACK=$p timeout 900 python bench.py --config c5 --steps 8 --warmup 2 --validate 0 --no-cpu-baseline > gpurun_out/xf/c5_p${p}.json 2> gpurun_out/xf/c5_p${p}.err
done
for f in gpurun_out/xf/*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"; done
