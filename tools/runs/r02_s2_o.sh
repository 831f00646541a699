timeout 600 python -m pytest tests/test_gpu_multigpu.py -q -x > gpurun_out/gt_o_multi.txt 2>&1; echo multi rc=$?; tail -2 gpurun_out/gt_o_multi.txt
V='{"default": {}, "contig": {"BLEST_DENSE_MIN": "1000000000"}, "tail4": {"BLEST_TAIL_DIV": "4"}}'
for c in c2 c3; do
timeout 600 python tools/ab.py --config $c --sources 8 --rounds 2 --levels --variants "$V" > gpurun_out/abo_$c.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/abo_$c.json'))
for k,v in d['variants'].items(): print('$c',k,v['ms_mean'],v['gteps_hm'],[(l['level'],l['s1_us']) for l in v['levels']])"
done
for G in 1 8; do timeout 600 python tools/rows_profile.py --config c2 --ranks $G --sources 1 > gpurun_out/rows_prof_$G.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/rows_prof_$G.json'))
for r in d['runs']: print('G=$G', r['total_us'], r['queue_per_rank'], [(l['level'],l['stage1_us'],l['exch_us'],l['sweep_us']) for l in r['levels']])"; done
