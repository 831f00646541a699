timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multigpu.py -m gpu -q -x > gpurun_out/gt_3a.txt 2>&1; echo tests rc=$?; tail -1 gpurun_out/gt_3a.txt
V='{"x": {}}'
for c in c4 c2 c1; do for lib in new prev new prev; do
  if [ $lib = new ]; then unset BLEST_LIB; else export BLEST_LIB=variants/$lib/libblest_b200.so; fi
  timeout 900 python tools/ab.py --config $c --sources 4 --rounds 2 --variants "$V" > gpurun_out/ab3a.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab3a.json'));v=d['variants']['x'];print('$c','$lib',v['ms_mean'],v['gteps_hm'])"
done; done
