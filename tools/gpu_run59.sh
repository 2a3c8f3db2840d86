#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 300 python tools/solve_timing.py 1 2 3 4 --quick > gpurun_out/solve_timing.log 2>&1
LAP_FUSE_ZSUMS=0 LAP_FUSE_TRANSFERS=0 timeout 300 python tools/solve_timing.py 2 --quick > gpurun_out/solve_timing_nofuse.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
