#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python tools/pool_probe.py 2 > gpurun_out/pool2.log 2>&1
timeout 600 python tools/pool_probe.py 3 > gpurun_out/pool3.log 2>&1
timeout 600 python tools/setup_trace.py 3 > gpurun_out/setup_trace3.log 2>&1
timeout 600 python tools/setup_trace.py 4 > gpurun_out/setup_trace4.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
