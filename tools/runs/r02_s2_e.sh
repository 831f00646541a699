# kBatch 2/3/4 builds x tail A/B on C2; C3 default
V='{"default": {}, "tail0": {"BLEST_TAIL_DIV": "0"}, "tail4": {"BLEST_TAIL_DIV": "4"}}'
for lib in kb3 kb4 kb2 kb3 kb4; do
  if [ $lib = kb3 ]; then unset BLEST_LIB; else export BLEST_LIB=variants/$lib/libblest_b200.so; fi
  for c in c2 c3; do
  timeout 600 python tools/ab.py --config $c --sources 8 --rounds 2 --levels --variants "$V" > gpurun_out/abe_${c}_$lib.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/abe_${c}_$lib.json'))
for k,v in d['variants'].items(): print('$c','$lib',k,v['ms_mean'],v['gteps_hm'],[(l['level'],l['s1_us'],l['us']) for l in v['levels']][1:5])"
  done
done
