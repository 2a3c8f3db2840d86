#!/bin/bash
# GPU iteration: the whole GPU suite, smoke, setup traces, solve timings, bench cfg 4, sharded 1x1 NCCL bench.
O=gpurun_out/iter${TAG}; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for k in 4 3 2; do LAP_SETUP_TRACE=2 timeout 600 python tools/setup_trace.py $k > $O/setup_trace$k.log 2>&1; echo "cfg$k $(grep 'default stream rep 3' $O/setup_trace$k.log)" >> $O/summary.txt; done
timeout 300 python tools/solve_timing.py 2 3 4 --quick > $O/solve_timing.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --shard --config 2 --no-cpu --steps 5 --warmup 3 > $O/bench_shard.json 2> $O/bench_shard.err; echo "rc=$?" >> $O/bench_shard.err
