#!/bin/bash
mkdir -p gpurun_out
for sh in 0 1 2 3; do for k in 2 3 4; do LAP_GSHIFT=$sh timeout 600 python tools/setup_trace.py $k > gpurun_out/gs${sh}_$k.log 2>&1; done; done
LAP_GSHIFT=3 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "hierarchy_spmv" > gpurun_out/pytest_g1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g1.log
