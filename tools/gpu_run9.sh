#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
LAP_TAIL=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "hierarchy_spmv" > gpurun_out/pytest_tail.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tail.log
for k in 1 2 3 4; do timeout 300 python tools/prof_solve.py $k > gpurun_out/prof_solve_fused$k.log 2>&1; done
for c in 8 16; do LAP_TAIL=1 LAP_TAIL_CTAS=$c timeout 300 python tools/prof_solve.py 1 > gpurun_out/prof_solve_tail1_$c.log 2>&1; LAP_TAIL=1 LAP_TAIL_CTAS=$c timeout 300 python tools/prof_solve.py 2 > gpurun_out/prof_solve_tail2_$c.log 2>&1; done
timeout 600 python tools/solve_timing.py 1 2 3 4 --quick > gpurun_out/solve_timing9.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
