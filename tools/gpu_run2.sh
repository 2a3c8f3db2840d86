#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m "gpu" -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python tools/solve_timing.py 1 2 3 4 > gpurun_out/solve_timing.log 2>&1
timeout 300 python tools/prof_cheb.py 2 5 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'sell<3' -c 2 -o gpurun_out/prof_cheb2 python tools/prof_cheb.py 2 5 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full.log
