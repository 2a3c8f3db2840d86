#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python tools/solve_timing.py 2 3 4 > gpurun_out/solve_timing3.log 2>&1
for k in 3 4 2; do
timeout 300 python tools/prof_solve.py $k > gpurun_out/prof_solve_plain$k.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "solve/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_solve$k.csv python tools/prof_solve.py $k > gpurun_out/ncu_solve$k.log 2>&1
done
timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 1 -o gpurun_out/prof_cheb2 python tools/prof_solve.py 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 4 -o gpurun_out/prof_cheb3 python tools/prof_solve.py 3 > gpurun_out/ncu_full3.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full3.log
