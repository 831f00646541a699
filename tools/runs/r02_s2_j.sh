timeout 600 python -m pytest tests/test_gpu_multigpu.py -q -x > gpurun_out/gt_j_multi.txt 2>&1; echo multi rc=$?; tail -2 gpurun_out/gt_j_multi.txt
for G in 1 8; do timeout 600 python tools/rows_profile.py --config c2 --ranks $G > gpurun_out/rows_prof_$G.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/rows_prof_$G.json'));print('G=$G vss',d['vss'])
for r in d['runs']: print(r['total_us'], r['queue_per_rank'], [(l['level'],l['stage1_us'],l['exch_us'],l['sweep_us']) for l in r['levels']])"; done
timeout 1500 python bench.py --config c5 --virtual-ranks 8 --steps 8 --warmup 2 --validate 2 > gpurun_out/b_c5_v8.json 2> gpurun_out/b_c5_v8.err; echo c5v8 rc=$?; tail -3 gpurun_out/b_c5_v8.err; cat gpurun_out/b_c5_v8.json
nvidia-smi --query-gpu=memory.used --format=csv
