#!/bin/bash
# ncu --set full of the fused Chebyshev step (k_spmv<E_CHEB>) on the first
# aggregation level of cfg k (tools/prof_cheb.py), summarised as text.
O=gpurun_out/final; mkdir -p $O
for k in ${CFGS:-4 3}; do
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"^k_spmv$" -s 2 -c 1 -o /tmp/cheb$k python tools/prof_cheb.py $k 5 > $O/ncu_cheb$k.log 2>&1
python tools/ncu_summary.py /tmp/cheb$k.ncu-rep > $O/ncu_full_cheb_cfg$k.txt 2>&1
ncu -i /tmp/cheb$k.ncu-rep --page details --csv > $O/ncu_full_cheb_cfg${k}_details.csv 2>&1
done
