#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
LAP_GSHIFT=3 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "hierarchy_spmv" > gpurun_out/pytest_g1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g1.log
for k in 2 3 4; do timeout 600 python tools/setup_trace.py $k > gpurun_out/setup_trace$k.log 2>&1; done
LAP_SETUP_TRACE=1 timeout 600 python tools/setup_trace.py 4 > gpurun_out/setup_trace4_phases.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
