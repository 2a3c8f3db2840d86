#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not full_size" > gpurun_out/pytest_quick.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quick.log
timeout 300 python tools/prof_solve.py 2 > gpurun_out/p2.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "setup/" --set full --clock-control none --import-source on -k regex:"k_tv_sweep|k_vote_round|k_gal_emit|k_affinity|k_relabel_emit" -c 5 -o gpurun_out/ncu_setup_cfg2 python tools/prof_solve.py 2 > gpurun_out/ncu_s.log 2>&1
