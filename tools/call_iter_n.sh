#!/bin/bash
O=gpurun_out/iter${TAG}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_block.py tests/test_gpu_kcycle.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for k in 4 3 2; do timeout 300 python tools/prof_solve.py $k > $O/p$k.txt 2>&1; echo "cfg$k $(grep 'solve_ms' $O/p$k.txt) $(grep vcycle $O/p$k.txt)" >> $O/summary.txt; done
USE_GRAPHS=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "solve/" --csv --log-file $O/solve4_launches.csv python tools/prof_solve.py 4 > $O/solve4_ncu.log 2>&1
timeout 300 python tools/block_timing.py 4 > $O/block4.jsonl 2>&1
