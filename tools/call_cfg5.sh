mkdir -p gpurun_out/r2
LAP_SETUP_TRACE=1 timeout 1500 python tools/cfg5_run.py ${SCALE:-26} > gpurun_out/r2/cfg5_run${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/r2/cfg5_run${TAG}.log
tail -40 gpurun_out/r2/cfg5_run${TAG}.log
