#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/block_prof.py 2 4 > gpurun_out/bp.log 2>&1 && \
timeout 900 ncu --kernel-name regex:k_blk_spmv --launch-skip 40 --launch-count 2 --set full --clock-control none --import-source on -o gpurun_out/ncu_blk_spmv python tools/block_prof.py 2 4 > gpurun_out/ncu_blk.log 2>&1
timeout 300 python tools/ktail_prof.py 2 > gpurun_out/kp.log 2>&1 && \
timeout 600 ncu --kernel-name regex:k_ktail --launch-skip 4 --launch-count 1 --set full --clock-control none --import-source on -o gpurun_out/ncu_ktail_final python tools/ktail_prof.py 2 > gpurun_out/ncu_kt.log 2>&1
