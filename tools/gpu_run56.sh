#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --kernel-name-base demangled --kernel-name regex:"k_blk_spmv<.int.0, .int.4>" --launch-skip 3 --launch-count 1 --set full --clock-control none --import-source on -o gpurun_out/ncu_blk_spmv_l0 python tools/block_prof.py 2 4 > gpurun_out/ncu_blk.log 2>&1
timeout 900 ncu --kernel-name-base demangled --kernel-name regex:"k_blk_spmv<.int.0, .int.8>" --launch-skip 3 --launch-count 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -o gpurun_out/ncu_blk_spmv_l0_k8 python tools/block_prof.py 2 8 > gpurun_out/ncu_blk8.log 2>&1
