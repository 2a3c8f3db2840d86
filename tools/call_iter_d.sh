#!/bin/bash
# GPU iteration: bit-exact parity (small + full-size), setup traces cfg 4 / 3 / 2.
O=gpurun_out/iter${TAG}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for k in 4 3 2; do LAP_SETUP_TRACE=2 timeout 600 python tools/setup_trace.py $k > $O/setup_trace$k.log 2>&1; done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "setup2/" -k regex:"$NCU" -c ${NK:-8} -o /tmp/setup_ncu python tools/prof_setup.py 4 > $O/ncu_setup.log 2>&1
ncu -i /tmp/setup_ncu.ncu-rep --page details --csv > $O/ncu_setup_details.csv 2>&1
fi
