#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/prof_solve.py 2 > gpurun_out/p2.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "setup/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_setup2.csv python tools/prof_solve.py 2 > gpurun_out/ncu_s2.log 2>&1
