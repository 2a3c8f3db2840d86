#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
timeout 900 python bench.py --no-cpu --no-clocks > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
timeout 900 python bench.py --no-cpu --steps 10 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
