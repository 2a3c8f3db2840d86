#!/bin/bash
mkdir -p gpurun_out
for k in 2 3 4; do
timeout 300 python tools/prof_solve.py $k > gpurun_out/prof_setup_plain$k.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "setup/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_setup$k.csv python tools/prof_solve.py $k > gpurun_out/ncu_setup$k.log 2>&1
done
