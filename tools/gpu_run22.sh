#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 600 python tools/solve_timing.py 1 2 3 4 --quick > gpurun_out/solve_timing22.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for k in 1 3 4; do timeout 900 python bench.py --config $k --no-cpu > gpurun_out/bench_cfg$k.json 2> gpurun_out/bench_cfg$k.err; done
