#!/bin/bash
# active-list vote rounds: GPU suite (hierarchies bit-exact vs the oracle, virtual
# grids, NCCL 1x1), bench cfg 4 / 3 / 2, warm setup phase trace of cfg 4
O=gpurun_out/votes; mkdir -p $O
export LAPGEN_CACHE=/tmp/lapgen_cache
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for k in 4 3 2; do timeout 600 python bench.py --config $k --no-cpu --steps 10 --warmup 3 > $O/bench_cfg$k.json 2> $O/bench_cfg$k.err; echo "rc=$?" >> $O/bench_cfg$k.err; done
LAP_SETUP_TRACE=2 timeout 600 python tools/setup_trace.py 4 > $O/setup_trace4.log 2>&1
