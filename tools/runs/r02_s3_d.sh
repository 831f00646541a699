V='{"x": {}, "nopf": {"BLEST_XFLAGS": "4096"}}'
for c in c4 c1; do for lib in new prev new; do
  if [ $lib = new ]; then unset BLEST_LIB; VV="$V"; else export BLEST_LIB=variants/$lib/libblest_b200.so; VV='{"x": {}}'; fi
  timeout 900 python tools/ab.py --config $c --sources 4 --rounds 2 --variants "$VV" > gpurun_out/ab3d.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/ab3d.json'))
for k,v in d['variants'].items(): print('$c','$lib',k,v['ms_mean'],v['gteps_hm'])"
done; done
