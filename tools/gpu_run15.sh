#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
for k in 1 2; do
  LAP_TAIL=0 timeout 300 python tools/prof_solve.py $k > gpurun_out/tail_off$k.log 2>&1
  timeout 300 python tools/prof_solve.py $k > gpurun_out/tail_8_$k.log 2>&1
  LAP_TAIL_CTAS=16 timeout 300 python tools/prof_solve.py $k > gpurun_out/tail_16_$k.log 2>&1
  LAP_TAIL_CTAS=4 timeout 300 python tools/prof_solve.py $k > gpurun_out/tail_4_$k.log 2>&1
done
timeout 600 python tools/solve_timing.py 1 2 3 4 --quick > gpurun_out/solve_timing15.log 2>&1
