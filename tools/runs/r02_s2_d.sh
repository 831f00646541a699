# lean stage-1 (sentinel word, no predicated moves): parity subset, then new vs head build, interleaved
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/gt_d.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/gt_d.txt
V='{"default": {}}'
for c in c2 c3; do
 for lib in new head new head; do
  if [ $lib = head ]; then export BLEST_LIB=variants/head/libblest_b200.so; else unset BLEST_LIB; fi
  timeout 600 python tools/ab.py --config $c --sources 8 --rounds 2 --levels --variants "$V" > gpurun_out/abd_${c}_$lib.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/abd_${c}_$lib.json'));v=d['variants']['default'];print('$c','$lib',v['ms_mean'],v['gteps_hm'],[(l['level'],l['s1_us'],l['us']) for l in v['levels']])"
 done
done
unset BLEST_LIB
