V='{"sigma": {}, "nosigma": {"BLEST_SIGMA": "0"}}'
timeout 600 python tools/ab.py --config c2 --sources 6 --rounds 2 --levels --variants "$V" > gpurun_out/abi_c2.json 2>gpurun_out/abi_c2.err
python -c "
import json;d=json.load(open('gpurun_out/abi_c2.json'))
for k,v in d['variants'].items(): print(k,v['ms_mean'],v['gteps_hm'],[(l['level'],l['queue'],l['s1_us'],l['us']) for l in v['levels']])"
