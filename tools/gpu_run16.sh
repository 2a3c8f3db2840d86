#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/solve_timing.py 3 4 2 --quick > gpurun_out/solve_timing16.log 2>&1
timeout 600 python tools/solve_timing.py 3 --quick >> gpurun_out/solve_timing16.log 2>&1
timeout 300 python tools/prof_solve.py 3 > gpurun_out/p3.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,power.draw --format=csv >> gpurun_out/solve_timing16.log
