mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "column_tiled or xt" > gpurun_out/r2/pytest_xt${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_xt${TAG}.log
tail -2 gpurun_out/r2/pytest_xt${TAG}.log
for k in 4 3; do timeout 600 python tools/prof_solve.py $k > gpurun_out/r2/levels_p$k${TAG}.txt 2>&1; done
grep -v "^\[" gpurun_out/r2/levels_p4${TAG}.txt | tail -9
