#!/bin/bash
# setup time of cfg 4 / 3 / 2 under lanes-per-row choices of the affinity / vote passes
O=gpurun_out/gsweep${TAG}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "hierarchy or full_size or memory_lean" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for k in 4 3 2; do
  for vg in 0 2 4 8; do for ag in 0 4 8; do
    LAP_VOTE_G=$vg LAP_AFF_G=$ag LAP_SETUP_TRACE=2 timeout 300 python tools/setup_trace.py $k > $O/t_${k}_v${vg}_a${ag}.log 2>&1
    echo "cfg$k vote_g=$vg aff_g=$ag $(grep 'default stream rep 3' $O/t_${k}_v${vg}_a${ag}.log)" >> $O/summary.txt
  done; done
done
