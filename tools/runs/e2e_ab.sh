# e2e leg variants: chunk size and pinned vs pageable output; host widening throughput probe
mkdir -p gpurun_out/e2
./tools/probes/widen_probe > gpurun_out/e2/widen_probe.txt 2>&1; cat gpurun_out/e2/widen_probe.txt
for i in 1 2; do
  for v in "16" "64" "64 --e2e-pageable" "16 --e2e-pageable"; do
    tag=$(echo $v | tr -d ' -')
    timeout 600 python bench.py --steps 64 --warmup 3 --validate 0 --no-cpu-baseline --e2e-chunk $v > gpurun_out/e2/c2_${tag}_$i.json 2> gpurun_out/e2/c2_${tag}_$i.err
  done
done
for v in "8" "8 --e2e-pageable"; do
  tag=$(echo $v | tr -d ' -')
  timeout 900 python bench.py --config c5 --steps 8 --warmup 2 --validate 0 --no-cpu-baseline --e2e-chunk $v > gpurun_out/e2/c5_${tag}.json 2> gpurun_out/e2/c5_${tag}.err
done
for f in gpurun_out/e2/*.json; do echo $f $(python -c "import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'])"); done
