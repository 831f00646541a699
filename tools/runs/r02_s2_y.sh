timeout 900 python -m pytest tests/test_gpu_multigpu.py -m gpu -q -x > gpurun_out/gt_y.txt 2>&1; echo tests rc=$?; tail -2 gpurun_out/gt_y.txt
for c in c2 c5; do timeout 900 python tools/rows_profile.py --config $c --ranks 8 --sources 1 > gpurun_out/rows_prof_y.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/rows_prof_y.json'))
for r in d['runs']: print('$c rows8', r['total_us'], [(l['level'],l['stage1_us'],l['exch_us'],l['sweep_us']) for l in r['levels']])"; done
