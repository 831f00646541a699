# masked row loads: parity subset + same-process A/B on C2 and C3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -k "lazy or c2 or c3 or variants or families" > gpurun_out/gt_c.txt 2>&1; echo pytest rc=$?; tail -3 gpurun_out/gt_c.txt
V='{"masked": {}, "plain": {"BLEST_XFLAGS": "128"}}'
timeout 900 python tools/ab.py --config c2 --sources 8 --rounds 3 --levels --variants "$V" > gpurun_out/ab_c2.json 2> gpurun_out/ab_c2.err; echo ab rc=$?; tail -2 gpurun_out/ab_c2.err
timeout 900 python tools/ab.py --config c3 --sources 8 --rounds 3 --levels --variants "$V" > gpurun_out/ab_c3.json 2> gpurun_out/ab_c3.err; echo ab rc=$?; tail -2 gpurun_out/ab_c3.err
python - <<'P'
import json
for c in ("c2","c3"):
    try: d=json.load(open(f"gpurun_out/ab_{c}.json"))
    except Exception as e: print(c, e); continue
    for k,v in d["variants"].items():
        print(c, k, v["ms_mean"], v["ms_round_means"], v["gteps_hm"])
        print("   ", [(l["level"], l["queue"], l["s1_us"], l["us"]) for l in v.get("levels", [])])
P
