for x in 1 2 3 0; do BLEST_XSTAMP=$x timeout 900 python tools/rows_profile.py --config c5 --ranks 8 --sources 1 > gpurun_out/rows_prof_z.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/rows_prof_z.json'))
r=d['runs'][0]; print('xstamp $x', r['total_us'], [(l['level'],l['exch_us']) for l in r['levels']])"; done
