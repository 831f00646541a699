#!/bin/bash
# C++ façade program (incl. the row-partitioned RowsEngine / rows_bfs_stepped block) on the B200
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cpp_facade.py -q -m gpu -x > gpurun_out/facade.txt 2>&1; echo "facade rc=$?"
tail -3 gpurun_out/facade.txt
