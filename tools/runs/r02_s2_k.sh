# ncu: rows kernel (1 virtual rank) vs the lazy kernel without the σ view, C2, one BFS each
M=lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:k_bfs_rows -s 1 -c 1 -o gpurun_out/ncu_rows1 python tools/rows_profile.py --config c2 --ranks 1 --sources 1 > gpurun_out/ncu_rows1.log 2>&1; echo rows rc=$?
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:k_bfs_lazy -s 2 -c 1 -o gpurun_out/ncu_lazy_nosig env BLEST_SIGMA=0 python tools/ab.py --config c2 --sources 1 --rounds 1 --variants '{"x": {}}' > gpurun_out/ncu_lazy.log 2>&1; echo lazy rc=$?
timeout 1200 python -m pytest tests/test_gpu_orderings.py -q -x -s -k "rcm" > gpurun_out/gt_rcm.txt 2>&1; echo rcm rc=$?; grep -E "GPU rcm|passed|failed|Error" gpurun_out/gt_rcm.txt | head
ls -la gpurun_out/*.ncu-rep
