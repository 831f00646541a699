# full gpu suite + default bench C2 (driver-equivalent) + C3/C4 bench lines
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gt_p.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/gt_p.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bp_c2.json 2> gpurun_out/bp_c2.err; echo c2 rc=$?; tail -2 gpurun_out/bp_c2.err
python -c "import json;d=json.load(open('gpurun_out/bp_c2.json'));print('c2',d['value'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['parity']['mismatches'],d['clocks'])"
timeout 900 python bench.py --config c3 --steps 16 --warmup 3 --validate 4 > gpurun_out/bp_c3.json 2> gpurun_out/bp_c3.err; echo c3 rc=$?
python -c "import json;d=json.load(open('gpurun_out/bp_c3.json'));print('c3',d['value'],d['ms_per_step'],d['roofline']['frac'],d['config']['prep_s'],d['parity']['mismatches'])"
timeout 1500 python bench.py --config c4 --steps 8 --warmup 3 --validate 2 > gpurun_out/bp_c4.json 2> gpurun_out/bp_c4.err; echo c4 rc=$?
python -c "import json;d=json.load(open('gpurun_out/bp_c4.json'));print('c4',d['value'],d['ms_per_step'],d['roofline']['frac'],d['config']['prep_s'],d['parity']['mismatches'])"
