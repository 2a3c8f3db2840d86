#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for k in 2 3 4; do
  timeout 300 python tools/prof_solve.py $k > gpurun_out/p${k}_fuse.log 2>&1
  LAP_FUSE_TRANSFERS=0 timeout 300 python tools/prof_solve.py $k > gpurun_out/p${k}_nofuse.log 2>&1
done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "full_size" > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
