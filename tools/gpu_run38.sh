#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kcycle.py -x -q -p no:cacheprovider > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size and not kcycle" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python tools/kcycle_timing.py > gpurun_out/kcycle_timing.log 2>&1
