timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/gt_x.txt 2>&1; echo tests rc=$?; tail -2 gpurun_out/gt_x.txt
V='{"x": {}}'
for c in c2 c5; do for lib in new prev new prev; do
  if [ $lib = new ]; then unset BLEST_LIB; else export BLEST_LIB=variants/$lib/libblest_b200.so; fi
  timeout 900 python tools/ab.py --config $c --sources 6 --rounds 2 --levels --variants "$V" > gpurun_out/abx.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/abx.json'));v=d['variants']['x'];print('$c','$lib',v['ms_mean'],v['gteps_hm'],[(l['level'],l['s1_us'],l['us']) for l in v['levels']])"
done; done
unset BLEST_LIB
timeout 900 python tools/rows_profile.py --config c5 --ranks 8 --sources 1 > gpurun_out/rows_prof_c5x.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/rows_prof_c5x.json'))
for r in d['runs']: print('c5 rows8', r['total_us'], [(l['level'],l['stage1_us'],l['exch_us'],l['sweep_us']) for l in r['levels']])"
