#!/bin/bash
mkdir -p gpurun_out
PROF_LEVEL=2 timeout 300 python tools/prof_solve.py 2 > gpurun_out/p2l2.log 2>&1 && PROF_LEVEL=2 timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 1 -o gpurun_out/ncu_cheb_cfg2_l2 python tools/prof_solve.py 2 > gpurun_out/ncu_l2.log 2>&1
