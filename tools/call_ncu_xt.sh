mkdir -p gpurun_out/r2
python tools/prof_cheb.py 3 3 > gpurun_out/r2/prof_cheb3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv_xt -s 2 -c 1 -o gpurun_out/r2/xt_prof python tools/prof_cheb.py 3 3 > gpurun_out/r2/ncu_xt.log 2>&1
tail -3 gpurun_out/r2/ncu_xt.log
