mkdir -p gpurun_out/r2
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/r2/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_gpu.log
tail -3 gpurun_out/r2/pytest_gpu.log
