#!/bin/bash
# End-of-round evidence on one B200 (profiles/r02/final_*): the GPU suite,
# smoke, bench lines (cfg 4 default + reference arm, cfg 2 / 3 / 5), per-level
# timings, setup traces, the ncu launch list of a short bench run, and one
# ncu --set full capture of the dominant kernel (cfg 4 level-0 Chebyshev step)
# and of cfg 3's level-1 step, summarised as text (the reports are not kept).
O=gpurun_out/final; mkdir -p $O
export LAPGEN_CACHE=/tmp/lapgen_cache
nvidia-smi > $O/nvidia_smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "rc=$?" >> $O/bench_cfg4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
for k in 2 3; do timeout 600 python bench.py --config $k --no-cpu --steps 10 --warmup 3 > $O/bench_cfg$k.json 2> $O/bench_cfg$k.err; echo "rc=$?" >> $O/bench_cfg$k.err; done
for k in 4 3 2; do timeout 600 python tools/prof_solve.py $k > $O/levels_p$k.txt 2>&1; done
for k in 4 3 2; do LAP_SETUP_TRACE=2 timeout 600 python tools/setup_trace.py $k > $O/setup_trace$k.log 2>&1; done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file /tmp/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launch.log 2>&1; gzip -c /tmp/launches.csv > $O/launches_bench_cfg4.csv.gz
CFGS="4 3" bash tools/call_ncu_cheb.sh
timeout 1200 python bench.py --config 5 --no-cpu --steps 3 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "rc=$?" >> $O/bench_cfg5.err
du -sh $O
