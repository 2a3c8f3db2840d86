#!/bin/bash
O=gpurun_out/iter${TAG}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_block.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for k in 4 3 2; do
LAP_SETUP_TRACE=2 timeout 300 python tools/setup_trace.py $k > $O/t$k.log 2>&1
echo "cfg$k $(grep 'default stream rep 3' $O/t$k.log)" >> $O/summary.txt
timeout 300 python tools/prof_solve.py $k > $O/p$k.txt 2>&1
echo "   $(grep 'solve_ms' $O/p$k.txt) $(grep 'level 1 kind' $O/p$k.txt) $(grep 'vcycle' $O/p$k.txt)" >> $O/summary.txt
done
