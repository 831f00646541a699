#!/bin/bash
# small stage 2 (dirty-word log on sparse lazy levels): parity, then same-process A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_orderings.py -m gpu -x -q > gpurun_out/ss_par.txt 2>&1; echo "par rc=$?"; tail -2 gpurun_out/ss_par.txt
for c in c2 c3 c5; do
timeout 900 python tools/ab.py --config $c --sources 8 --rounds 3 --levels --variants '{"small": {}, "sweep": {"BLEST_SMALL_S2": "0"}}' > gpurun_out/ss_ab_$c.json 2> gpurun_out/ss_ab_$c.err
python - $c <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/ss_ab_{sys.argv[1]}.json"))
for k, v in d["variants"].items():
    print(sys.argv[1], k, v["ms_mean"], v["gteps_hm"], v["ms_round_means"], [(l["level"], l["queue"], l["s1_us"], l["us"]) for l in v.get("levels", [])][:12])
PY
done
for lib in variants/base/libblest_b200.so paper_2512_21967_b200/libblest_b200.so; do
BLEST_LIB=$lib timeout 900 python bench.py --config c2 --steps 32 --no-cpu-baseline --validate 4 > gpurun_out/ss_b.json 2> gpurun_out/ss_b.err
python -c "import json;d=json.load(open('gpurun_out/ss_b.json'));print('$lib', d['value'], d['ms_per_step'], d['roofline']['frac'], d['parity']['mismatches'])"
done
