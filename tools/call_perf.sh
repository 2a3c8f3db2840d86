mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=30 -k "import or dist or full_size" > gpurun_out/r2/pytest_gpu${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_gpu${TAG}.log
tail -3 gpurun_out/r2/pytest_gpu${TAG}.log
for k in 4 3; do timeout 600 python tools/prof_solve.py $k > gpurun_out/r2/levels_p$k${TAG}.txt 2>&1; done
CFGS="4 3" bash tools/call_trace.sh
