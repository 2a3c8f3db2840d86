#!/bin/bash
mkdir -p gpurun_out
for r in 1 2; do timeout 300 python tools/solve_timing.py 1 2 3 4 --quick; done > gpurun_out/solve_timing.log 2>&1
timeout 300 python tools/prof_solve.py 1 > gpurun_out/p1.log 2>&1
