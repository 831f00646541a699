timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_cpp_facade.py -m gpu -q -x > gpurun_out/gt_t.txt 2>&1; echo parity rc=$?; tail -2 gpurun_out/gt_t.txt
V='{"x": {}}'
for c in c2 c3; do for lib in new prev new prev; do
  if [ $lib = new ]; then unset BLEST_LIB; else export BLEST_LIB=variants/$lib/libblest_b200.so; fi
  timeout 600 python tools/ab.py --config $c --sources 10 --rounds 2 --levels --variants "$V" > gpurun_out/abt.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/abt.json'));v=d['variants']['x'];print('$c','$lib',v['ms_mean'],v['gteps_hm'],[(l['level'],l['s1_us'],l['us']) for l in v['levels']])"
done; done
