#!/bin/bash
# Quick GPU check during development (gpurun): GPU tests without the full-size
# parity cases, then solve timings of cfg 1-4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 300 python tools/solve_timing.py 1 2 3 4 --quick > gpurun_out/solve_timing.log 2>&1
