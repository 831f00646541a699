V='{"x": {}, "nosig": {"BLEST_SIGMA": "0"}}'
for lib in new minb3; do
  if [ $lib = new ]; then unset BLEST_LIB; else export BLEST_LIB=variants/$lib/libblest_b200.so; fi
  for c in c3 c2; do
  timeout 600 python tools/ab.py --config $c --sources 8 --rounds 2 --levels --variants "$V" > gpurun_out/abv.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/abv.json'))
for k,v in d['variants'].items(): print('$c','$lib',k,v['ms_mean'],v['gteps_hm'],[(l['level'],l['s1_us'],l['us']) for l in v['levels']])"
done; done
unset BLEST_LIB
for k in 1 2 3; do timeout 900 python bench.py --steps 32 --warmup 5 --validate 0 --no-cpu-baseline > gpurun_out/bv_c2.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/bv_c2.json'));print('c2',d['value'],d['roofline']['frac'],d['e2e']['value'])"; done
