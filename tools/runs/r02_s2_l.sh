for G in 1 8; do timeout 600 python tools/rows_profile.py --config c2 --ranks $G > gpurun_out/rows_prof_$G.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/rows_prof_$G.json'));print('G=$G vss',d['vss'])
for r in d['runs']: print(r['total_us'], r['queue_per_rank'], [(l['level'],l['stage1_us'],l['exch_us'],l['sweep_us']) for l in r['levels']])"; done
