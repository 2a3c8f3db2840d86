#!/bin/bash
mkdir -p gpurun_out
for v in "A=1" "LAP_FUSE_ZSUMS=0" "LAP_FUSE_TRANSFERS=0" "LAP_FUSE_ZSUMS=0 LAP_FUSE_TRANSFERS=0"; do
  for r in 1 2; do echo "$v: $(env $v timeout 300 python tools/solve_timing.py 2 --quick 2>&1 | tail -1)"; done
done > gpurun_out/fuse_ab.log
