# evidence after the lazy dense threshold: tests, bench c2 x2, ncu (launch list + full capture with atomic/RED sectors), phase timeline
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gt_r.txt 2>&1; echo pytest rc=$?; tail -2 gpurun_out/gt_r.txt
for k in 1 2; do timeout 900 python bench.py --steps 64 --warmup 5 --validate 20 > gpurun_out/br_c2_$k.json 2> gpurun_out/br_c2_$k.err; echo c2 rc=$?
python -c "import json;d=json.load(open('gpurun_out/br_c2_$k.json'));print('c2',d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['parity']['checked'],d['parity']['mismatches'],d['clocks']['sm_mhz'])"; done
timeout 600 python tools/phase_profile.py --config c2 --sources 2 > gpurun_out/r02_phase_c2.txt 2>&1
timeout 1200 bash tools/profile.sh c2 > gpurun_out/profile_c2.log 2>&1; echo prof rc=$?
ls -la gpurun_out/full_c2.ncu-rep gpurun_out/launches_c2.csv
