#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for k in 1 2 3 4; do timeout 300 python tools/prof_solve.py $k > gpurun_out/dt_$k.log 2>&1; LAP_DENSE_TAIL=0 timeout 300 python tools/prof_solve.py $k > gpurun_out/dt_off_$k.log 2>&1; done
timeout 600 python tools/solve_timing.py 1 2 3 4 --quick > gpurun_out/solve_timing21.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
