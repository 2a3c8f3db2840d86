mkdir -p gpurun_out/r2
for k in ${CFGS:-4 3}; do
LAP_SETUP_TRACE=1 timeout 600 python tools/setup_trace.py $k > gpurun_out/r2/setup_trace$k.log 2>&1
done
