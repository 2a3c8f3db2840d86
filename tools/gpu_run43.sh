#!/bin/bash
mkdir -p gpurun_out
LAP_KTAIL_INFO=1 timeout 300 python tools/ktail_prof.py 2 > gpurun_out/ktail_info2.log 2>&1
LAP_KTAIL_INFO=1 timeout 300 python tools/ktail_prof.py 1 > gpurun_out/ktail_info1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kcycle.py -x -q -p no:cacheprovider > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 900 python tools/kcycle_timing.py cfg1 cfg2 cfg3 cfg4 grid2d_1024 > gpurun_out/kcycle_timing.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ktail_launches2.csv python tools/ktail_prof.py 2 > gpurun_out/ncu_ktail_l.log 2>&1
