#!/bin/bash
mkdir -p gpurun_out
LAP_KTAIL_TRACE=1 LAP_KTAIL_INFO=1 timeout 300 python tools/ktail_prof.py 2 > gpurun_out/ktail_trace2.log 2>&1
LAP_KTAIL_TRACE=1 LAP_KTAIL_INFO=1 timeout 300 python tools/ktail_prof.py 1 > gpurun_out/ktail_trace1.log 2>&1
