#!/bin/bash
mkdir -p gpurun_out
LAP_KTAIL_TRACE=1 LAP_KTAIL_INFO=1 timeout 300 python tools/ktail_prof.py 2 > gpurun_out/ktail_trace2.log 2>&1
LAP_KTAIL_TRACE=1 LAP_KTAIL_INFO=1 timeout 300 python tools/ktail_prof.py 1 > gpurun_out/ktail_trace1.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kcycle.py -x -q -p no:cacheprovider > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 900 python tools/kcycle_timing.py cfg1 cfg2 grid2d_1024 > gpurun_out/kcycle_timing.log 2>&1
