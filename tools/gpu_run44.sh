#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --kernel-name regex:k_ktail --set full --clock-control none --import-source on -c 1 -o gpurun_out/ncu_ktail3 python tools/ktail_prof.py 2 > gpurun_out/ncu_ktail.log 2>&1
