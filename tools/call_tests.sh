mkdir -p gpurun_out/r2
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/r2/pytest_gpu${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/r2/pytest_gpu${TAG}.log
tail -3 gpurun_out/r2/pytest_gpu${TAG}.log
