#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q -p no:cacheprovider > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size and not sharded and not replication" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
