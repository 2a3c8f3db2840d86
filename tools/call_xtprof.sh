mkdir -p gpurun_out/r2
python tools/prof_xt.py > gpurun_out/r2/prof_xt${TAG}.log 2>&1
LAP_XT=0 python tools/prof_xt.py > gpurun_out/r2/prof_xt_off${TAG}.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "column_tiled or xt" > gpurun_out/r2/pytest_xt${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_xt${TAG}.log
cat gpurun_out/r2/prof_xt${TAG}.log gpurun_out/r2/prof_xt_off${TAG}.log; tail -2 gpurun_out/r2/pytest_xt${TAG}.log
