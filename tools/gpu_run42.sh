#!/bin/bash
mkdir -p gpurun_out
LAP_KTAIL_INFO=1 timeout 300 python tools/ktail_prof.py 2 > gpurun_out/ktail_info2.log 2>&1
LAP_KTAIL_INFO=1 timeout 300 python tools/ktail_prof.py 1 > gpurun_out/ktail_info1.log 2>&1
timeout 600 ncu --kernel-name regex:k_ktail --set full --clock-control none --import-source on -c 2 -o gpurun_out/ncu_ktail2 python tools/ktail_prof.py 2 > gpurun_out/ncu_ktail.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ktail_launches2.csv python tools/ktail_prof.py 2 > gpurun_out/ncu_ktail_l.log 2>&1
