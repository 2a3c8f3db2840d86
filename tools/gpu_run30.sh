#!/bin/bash
mkdir -p gpurun_out
LAP_SETUP_TRACE=1 timeout 600 python tools/setup_trace.py 4 > gpurun_out/setup_trace4_phases.log 2>&1
