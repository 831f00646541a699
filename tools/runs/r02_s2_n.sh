for env in "X=1" "BLEST_DENSE_MIN=1" "BLEST_DENSE_MIN=1000000000" "BLEST_TAIL_DIV=2"; do
env $env timeout 600 python tools/rows_profile.py --config c2 --ranks 1 --sources 1 > gpurun_out/rp.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/rp.json'))
for r in d['runs']: print('$env', r['total_us'], [(l['level'],l['stage1_us']) for l in r['levels']])"
done
