#!/bin/bash
# storage row-sort threshold: setup time and per-level solve times on cfg 4 / 3
O=gpurun_out/sortmax; mkdir -p $O
for sm in 64 2048 100000000; do for k in 4 3; do
LAP_SORT_MAX=$sm LAP_SETUP_TRACE=2 timeout 300 python tools/setup_trace.py $k > $O/t${k}_$sm.log 2>&1
echo "cfg$k sort_max=$sm $(grep 'default stream rep 3' $O/t${k}_$sm.log)" >> $O/summary.txt
LAP_SORT_MAX=$sm timeout 300 python tools/prof_solve.py $k > $O/p${k}_$sm.txt 2>&1
echo "   $(grep 'solve_ms' $O/p${k}_$sm.txt) $(grep 'level 1 kind' $O/p${k}_$sm.txt) $(grep 'vcycle' $O/p${k}_$sm.txt)" >> $O/summary.txt
done; done
