timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/gt_w.txt 2>&1; echo tests rc=$?; tail -3 gpurun_out/gt_w.txt
V='{"auto": {}, "force": {"BLEST_SIGMA": "1"}}'
for c in c3 c2; do
timeout 600 python tools/ab.py --config $c --sources 8 --rounds 2 --variants "$V" > gpurun_out/abw.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/abw.json'))
for k,v in d['variants'].items(): print('$c',k,v['ms_mean'],v['gteps_hm'])"
done
for G in 1 8; do timeout 600 python tools/rows_profile.py --config c2 --ranks $G --sources 1 > gpurun_out/rows_prof_$G.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/rows_prof_$G.json'))
for r in d['runs']: print('G=$G', r['total_us'], r['queue_per_rank'], [(l['level'],l['stage1_us'],l['exch_us'],l['sweep_us']) for l in r['levels']])"; done
