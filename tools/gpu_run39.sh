#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kcycle.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 900 python tools/kcycle_timing.py cfg1 cfg2 cfg3 cfg4 grid2d_1024 > gpurun_out/kcycle_timing.log 2>&1
for k in 2 4; do timeout 300 python tools/prof_solve.py $k > gpurun_out/p${k}_fuse.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size and not kcycle and not parity" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
