#!/bin/bash
# Full round-end evidence refresh on one B200 (gpurun): GPU tests, bench lines for
# cfg 1-4 + the reference arm, solve timings, per-level timings, K-cycle and
# block timings, and the launch list of a short bench run.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_all.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for k in 1 3 4; do timeout 900 python bench.py --config $k --no-cpu > gpurun_out/bench_cfg$k.json 2> gpurun_out/bench_cfg$k.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/solve_timing.py 1 2 3 4 --quick > gpurun_out/solve_timing.log 2>&1
for k in 2 3 4; do timeout 300 python tools/prof_solve.py $k > gpurun_out/p$k.log 2>&1; done
timeout 900 python tools/kcycle_timing.py cfg1 cfg2 cfg3 cfg4 grid2d_1024 > gpurun_out/kcycle_timing.log 2>&1
timeout 900 python tools/block_timing.py > gpurun_out/block_timing.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
