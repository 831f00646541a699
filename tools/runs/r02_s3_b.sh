timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/gt_3b.txt 2>&1; echo tests rc=$?; tail -1 gpurun_out/gt_3b.txt
V='{"x": {}}'
for c in c2 c5; do for lib in new prev new prev; do
  if [ $lib = new ]; then unset BLEST_LIB; else export BLEST_LIB=variants/$lib/libblest_b200.so; fi
  timeout 900 python tools/ab.py --config $c --sources 6 --rounds 2 --levels --variants "$V" > gpurun_out/ab3b.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab3b.json'));v=d['variants']['x'];print('$c','$lib',v['ms_mean'],v['gteps_hm'],[(l['level'],round(l['us']-(l['s1_us'] or 0),1)) for l in v['levels']])"
done; done
