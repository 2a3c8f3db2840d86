#!/bin/bash
# Round-2 evidence on one B200: GPU tests, smoke, bench (cfg 4 default + cfg 2/3),
# the reference arm, per-level timings, and the launch list of a short bench run.
O=gpurun_out/r2${TAG}
mkdir -p $O
nvidia-smi > $O/nvidia_smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
for k in 2 3; do timeout 600 python bench.py --config $k --no-cpu --steps 10 --warmup 3 > $O/bench_cfg$k.json 2> $O/bench_cfg$k.err; done
for k in 4 3 2; do timeout 600 python tools/prof_solve.py $k > $O/levels_p$k.txt 2>&1; done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_bench.log 2>&1
