#!/bin/bash
# GPU iteration: bit-exact parity + dist setup tests, setup traces (default and
# long rows unsorted), solve timings with unsorted long rows.
O=gpurun_out/iter${TAG}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -x -k "hierarchy or full_size or memory_lean or distributed or pattern" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for k in 4 3 2; do LAP_SETUP_TRACE=2 timeout 600 python tools/setup_trace.py $k > $O/setup_trace$k.log 2>&1; echo "cfg$k default $(grep 'default stream rep 3' $O/setup_trace$k.log)" >> $O/summary.txt; done
for k in 4 3 2; do LAP_SORT_LONG=0 LAP_SETUP_TRACE=2 timeout 600 python tools/setup_trace.py $k > $O/setup_trace${k}_nosortlong.log 2>&1; echo "cfg$k nosortlong $(grep 'default stream rep 3' $O/setup_trace${k}_nosortlong.log)" >> $O/summary.txt; done
timeout 300 python tools/solve_timing.py 2 3 4 --quick > $O/solve_timing.log 2>&1
LAP_SORT_LONG=0 timeout 300 python tools/solve_timing.py 2 3 4 --quick > $O/solve_timing_nosortlong.log 2>&1
