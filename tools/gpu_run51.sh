#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py -x -q -p no:cacheprovider > gpurun_out/pytest_blk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_blk.log
timeout 900 python tools/block_timing.py > gpurun_out/block_timing.log 2>&1
