#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
for k in 1 3 4; do timeout 900 python bench.py --config $k --no-cpu > gpurun_out/bench_cfg$k.json 2> gpurun_out/bench_cfg$k.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python tools/prof_solve.py 2 > gpurun_out/p2.log 2>&1 && timeout 600 ncu --nvtx --nvtx-include "cheb/" --set full --clock-control none --import-source on -c 1 -o gpurun_out/ncu_cheb_cfg2_l0 python tools/prof_solve.py 2 > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "solve/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_solve2.csv python tools/prof_solve.py 2 > gpurun_out/ncu5.log 2>&1
