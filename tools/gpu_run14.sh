#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/prof_solve.py 2 > gpurun_out/p2.log 2>&1 && timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 1 -o gpurun_out/ncu_cheb_cfg2_l0 python tools/prof_solve.py 2 > gpurun_out/ncu1.log 2>&1
PROF_LEVEL=2 timeout 300 python tools/prof_solve.py 4 > gpurun_out/p4.log 2>&1 && PROF_LEVEL=2 timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 1 -o gpurun_out/ncu_cheb_cfg4_l2 python tools/prof_solve.py 4 > gpurun_out/ncu2.log 2>&1
timeout 300 python tools/prof_solve.py 3 > gpurun_out/p3.log 2>&1 && timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 1 -o gpurun_out/ncu_cheb_cfg3_l1 python tools/prof_solve.py 3 > gpurun_out/ncu3.log 2>&1
timeout 300 python tools/prof_solve.py 4 > gpurun_out/p4b.log 2>&1 && timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 1 -o gpurun_out/ncu_cheb_cfg4_l0 python tools/prof_solve.py 4 > gpurun_out/ncu4.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "solve/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_solve2.csv python tools/prof_solve.py 2 > gpurun_out/ncu5.log 2>&1
