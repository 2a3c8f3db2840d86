#!/bin/bash
# GPU iteration: parity (bit-exact hierarchy), distributed-setup and pattern-only
# tests, setup traces with the two canonical quantisers, an ncu capture of the
# setup's canonical SpMV / vote / affinity kernels (exported as text, the
# report itself not kept: gpurun_out is capped at 64 MiB), cfg 5 bench line.
export LAPGEN_CACHE=/tmp/lapgen_cache
O=gpurun_out/iter_c; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -x -k "not full_size" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for k in 4 3; do LAP_SETUP_TRACE=2 timeout 600 python tools/setup_trace.py $k > $O/setup_trace$k.log 2>&1; done
for k in 4 3; do LAP_CANON_Q=int LAP_SETUP_TRACE=2 timeout 600 python tools/setup_trace.py $k > $O/setup_trace${k}_int.log 2>&1; done
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "setup2/" -k regex:"k_cspmv_store|k_vote_round|k_affinity|k_normalize" -c 14 -o /tmp/setup_cfg4 python tools/prof_setup.py 4 > $O/ncu_setup_cfg4.log 2>&1
ncu -i /tmp/setup_cfg4.ncu-rep --page details --csv > $O/ncu_setup_cfg4_details.csv 2>&1
ncu -i /tmp/setup_cfg4.ncu-rep --page raw --csv > /tmp/raw.csv 2>&1; gzip -c /tmp/raw.csv > $O/ncu_setup_cfg4_raw.csv.gz
timeout 900 python bench.py --config 5 --no-cpu --steps 3 --warmup 3 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "rc=$?" >> $O/bench_cfg5.err
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "full_size" > $O/pytest_full.log 2>&1; echo "rc=$?" >> $O/pytest_full.log
du -sh $O
