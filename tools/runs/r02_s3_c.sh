V='{"x": {}, "pf": {"BLEST_XFLAGS": "2048"}}'
for c in c2 c3; do for lib in new prev new prev; do
  if [ $lib = new ]; then unset BLEST_LIB; VV="$V"; else export BLEST_LIB=variants/$lib/libblest_b200.so; VV='{"x": {}}'; fi
  timeout 900 python tools/ab.py --config $c --sources 6 --rounds 2 --variants "$VV" > gpurun_out/ab3c.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab3c.json'))
for k,v in d['variants'].items(): print('$c','$lib',k,v['ms_mean'],v['gteps_hm'])"
done; done
