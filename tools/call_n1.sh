#!/bin/bash
# N1 row-split passes on one B200: the GPU suite (virtual-grid and 1x1 NCCL
# distributed-setup tests), smoke, and cfg 4 / 3 bench lines (single-GPU path:
# no split) to check the setup time did not move.
O=gpurun_out/n1; mkdir -p $O
export LAPGEN_CACHE=/tmp/lapgen_cache
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=10 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "rc=$?" >> $O/bench_cfg4.err
timeout 600 python bench.py --config 3 --no-cpu --steps 10 --warmup 3 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "rc=$?" >> $O/bench_cfg3.err
