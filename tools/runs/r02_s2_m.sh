timeout 600 python tools/rows_profile.py --config c2 --ranks 1 --compare-lazy > gpurun_out/rows_prof_cmp.json 2>gpurun_out/rows_prof_cmp.err; tail -2 gpurun_out/rows_prof_cmp.err
python -c "
import json;d=json.load(open('gpurun_out/rows_prof_cmp.json'))
for r in d['runs']: print('rows', r['total_us'], [(l['level'],l['stage1_us'],l['exch_us'],l['sweep_us']) for l in r['levels']])
for k,v in d['lazy'].items():
  for r in v: print(k, r['total_us'], r['levels'])"
BLEST_TAIL_DIV=0 timeout 600 python tools/rows_profile.py --config c2 --ranks 1 --sources 1 > gpurun_out/rows_prof_t0.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/rows_prof_t0.json'))
for r in d['runs']: print('rows tail0', r['total_us'], [(l['level'],l['stage1_us'],l['exch_us'],l['sweep_us']) for l in r['levels']])"
