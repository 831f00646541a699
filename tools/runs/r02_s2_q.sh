V='{"dm38k": {}, "dm200k": {"BLEST_DENSE_MIN": "200000"}, "dm500k": {"BLEST_DENSE_MIN": "500000"}, "dm1m": {"BLEST_DENSE_MIN": "1000000"}, "dm2m": {"BLEST_DENSE_MIN": "2000000"}}'
for c in c2 c3; do
timeout 900 python tools/ab.py --config $c --sources 10 --rounds 2 --levels --variants "$V" > gpurun_out/abq_$c.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/abq_$c.json'))
for k,v in d['variants'].items(): print('$c',k,v['ms_mean'],v['ms_round_means'],v['gteps_hm'],[(l['level'],l['queue'],l['s1_us'],l['us']) for l in v['levels']])"
done
