#!/bin/bash
# One development iteration on the GPU: selected GPU tests, setup phase trace,
# block timings.  TESTS, CFGS, BLOCK_CFGS, BLOCK_KS from the environment.
O=gpurun_out/iter${TAG}
mkdir -p $O
if [ -n "$TESTS" ]; then
timeout 1200 python -m pytest $TESTS -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
fi
for k in ${CFGS}; do
LAP_SETUP_TRACE=2 timeout 600 python tools/setup_trace.py $k > $O/setup_trace$k.log 2>&1
done
if [ -n "$BLOCK_CFGS" ]; then
timeout 900 python tools/block_timing.py $BLOCK_CFGS > $O/block_timing.jsonl 2>&1
fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA" > $O/extra.log 2>&1; fi
