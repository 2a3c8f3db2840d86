#!/bin/bash
mkdir -p gpurun_out
LAP_PDL=0 timeout 300 python tools/prof_solve.py 2 > gpurun_out/prof_solve_nopdl2.log 2>&1
timeout 300 python tools/prof_solve.py 1 > gpurun_out/prof_solve_plain1.log 2>&1
LAP_PDL=0 timeout 300 python tools/prof_solve.py 1 > gpurun_out/prof_solve_nopdl1.log 2>&1
