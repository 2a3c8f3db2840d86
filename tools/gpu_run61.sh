#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for v in "A=1" "LAP_FUSE_TRANSFERS=0" "A=1" "LAP_FUSE_TRANSFERS=0"; do
  for c in 2 3 4; do echo "$v: $(env $v timeout 300 python tools/solve_timing.py $c --quick 2>&1 | tail -1)"; done
done > gpurun_out/fuse_ab.log
