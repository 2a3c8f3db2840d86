#!/bin/bash
# cfg 5 (R-MAT s26) evidence on one B200: the end-to-end run with the setup
# phase trace and per-level timings, the GPU parity test, and a bench line.
O=gpurun_out/cfg5${TAG}
mkdir -p $O
export LAPGEN_CACHE=/tmp/lapgen_cache
free -g > $O/free.txt; nproc >> $O/free.txt
LAP_SETUP_TRACE=1 REPS=2 timeout 1500 python tools/cfg5_run.py 26 > $O/cfg5_run.log 2>&1; echo "rc=$?" >> $O/cfg5_run.log
LAP_TEST_CFG5=1 timeout 1800 python -m pytest tests/test_gpu_cfg5.py -m gpu -q -p no:cacheprovider > $O/pytest_cfg5.log 2>&1; echo "rc=$?" >> $O/pytest_cfg5.log
timeout 1200 python bench.py --config 5 --no-cpu --steps 3 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "rc=$?" >> $O/bench_cfg5.err
