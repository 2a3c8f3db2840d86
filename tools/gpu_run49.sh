#!/bin/bash
mkdir -p gpurun_out
for t in 1024 512 256; do
LAP_KTAIL_THREADS=$t LAP_KTAIL_TRACE=1 timeout 300 python tools/ktail_prof.py 2 2>&1 | tail -2 | head -1 > gpurun_out/kt_thr_$t.log
LAP_KTAIL_THREADS=$t LAP_KTAIL_TRACE=1 timeout 300 python tools/ktail_prof.py 1 2>&1 | tail -2 | head -1 >> gpurun_out/kt_thr_$t.log
done
