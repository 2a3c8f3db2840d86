#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for r in 1 2; do timeout 300 python tools/solve_timing.py 1 2 3 4 --quick; done > gpurun_out/solve_timing.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "solve/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_solve2.csv python tools/prof_solve.py 2 > gpurun_out/ncu5.log 2>&1
