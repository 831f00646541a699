# full -m gpu suite (no -x: see every failure), with durations
timeout 3000 python -m pytest tests -m gpu -q --durations=25 -p no:cacheprovider > gpurun_out/gputest_s2b.txt 2>&1; echo pytest rc=$?; tail -45 gpurun_out/gputest_s2b.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo smoke rc=$?; tail -3 gpurun_out/smoke.txt
