#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for k in 2 3 4; do timeout 300 python tools/prof_solve.py $k > gpurun_out/ps_$k.log 2>&1; LAP_SORT_ROWS=0 timeout 300 python tools/prof_solve.py $k > gpurun_out/ps_nosort_$k.log 2>&1; done
timeout 600 python tools/solve_timing.py 1 2 3 4 --quick > gpurun_out/solve_timing34.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
