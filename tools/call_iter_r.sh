#!/bin/bash
O=gpurun_out/iter${TAG}; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for k in 4 3 2; do
LAP_SETUP_TRACE=2 timeout 300 python tools/setup_trace.py $k > $O/t$k.log 2>&1
echo "cfg$k $(grep 'default stream rep 3' $O/t$k.log)" >> $O/summary.txt
done
