#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for v in 0 3000000 8000000 20000000; do LAP_NB4_MAXNNZ=$v timeout 300 python tools/prof_solve.py 2 > gpurun_out/nb4_$v.log 2>&1; done
LAP_NB4_MAXNNZ=8000000 timeout 300 python tools/prof_solve.py 4 > gpurun_out/nb4_cfg4.log 2>&1
timeout 300 python tools/prof_solve.py 4 > gpurun_out/nb8_cfg4.log 2>&1
