# completion filter: parity variants, A/B (pre-CF build vs CF=0 vs CF=1); rows timeline G=1/8 on C2
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variants or families or dense" > gpurun_out/gt_h.txt 2>&1; echo parity rc=$?; tail -3 gpurun_out/gt_h.txt
timeout 600 python -m pytest tests/test_gpu_multigpu.py -q -x > gpurun_out/gt_h_multi.txt 2>&1; echo multi rc=$?; tail -2 gpurun_out/gt_h_multi.txt
V='{"cf0": {}, "cf1": {"BLEST_CF": "1"}}'
for c in c2 c3; do
 for lib in new precf new; do
  if [ $lib = new ]; then unset BLEST_LIB; VV="$V"; else export BLEST_LIB=variants/$lib/libblest_b200.so; VV='{"cf0": {}}'; fi
  timeout 600 python tools/ab.py --config $c --sources 8 --rounds 2 --levels --variants "$VV" > gpurun_out/abh_${c}_$lib.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/abh_${c}_$lib.json'))
for k,v in d['variants'].items(): print('$c','$lib',k,v['ms_mean'],v['gteps_hm'],[(l['level'],l['queue'],l['s1_us'],l['us']) for l in v['levels']])"
 done
done
unset BLEST_LIB
for G in 1 8; do timeout 600 python tools/rows_profile.py --config c2 --ranks $G > gpurun_out/rows_prof_$G.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/rows_prof_$G.json'));print('G=$G vss',d['vss'])
for r in d['runs']: print(r['total_us'], r['queue_per_rank'], [(l['level'],l['stage1_us'],l['exch_us'],l['sweep_us']) for l in r['levels']])"; done
