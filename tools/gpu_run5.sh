#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for k in 2 3 4; do timeout 300 python tools/prof_solve.py $k > gpurun_out/prof_solve_plain$k.log 2>&1; done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 1 -o gpurun_out/prof_cheb2 python tools/prof_solve.py 2 > gpurun_out/ncu_full2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full2.log
timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 1 -o gpurun_out/prof_cheb4 python tools/prof_solve.py 4 > gpurun_out/ncu_full4.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_full4.log
