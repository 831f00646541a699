export PYTHONFAULTHANDLER=1
timeout 300 python bench.py --config c1 --steps 4 --warmup 3 > gpurun_out/dbg.json 2> gpurun_out/dbg.err; echo rc=$?
tail -30 gpurun_out/dbg.err; cat gpurun_out/dbg.json
