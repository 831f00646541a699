#!/bin/bash
# ncu evidence for the bench workload (run under gpurun on one B200):
#   1. launch list of the bench command (every library kernel, device time per launch)
#   2. one --set full capture of a BFS launch (DRAM traffic, stalls, source attribution)
# Outputs in gpurun_out/; tools/summarize_profile.py turns them into profiles/*.
set -e
CFG=${1:-c2}
MODE=${2:-b200}
OUT=gpurun_out
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${CFG}.csv \
    python bench.py --config $CFG --mode $MODE --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/launches_${CFG}.log 2>&1 || true
ncu --set full --metrics lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_op_imma.sum,sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none --import-source on -k regex:k_bfs -s 3 -c 1 -o $OUT/full_${CFG} \
    python bench.py --config $CFG --mode $MODE --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/full_${CFG}.log 2>&1 || true
