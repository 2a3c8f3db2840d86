#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python tools/solve_timing.py 1 2 3 4 --quick > gpurun_out/solve_timing11.log 2>&1
for k in 3 4; do
timeout 300 python tools/prof_solve.py $k > gpurun_out/prof_setup_plain$k.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "setup/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_setup$k.csv python tools/prof_solve.py $k > gpurun_out/ncu_setup$k.log 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
