mkdir -p gpurun_out/r2
lscpu > gpurun_out/r2/lscpu.txt 2>&1; free -g >> gpurun_out/r2/lscpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/r2/bench${TAG}.json 2> gpurun_out/r2/bench${TAG}.err; echo "rc=$?" >> gpurun_out/r2/bench${TAG}.err
if [ -z "$NOREF" ]; then
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 ${BENCH_ARGS} > gpurun_out/r2/bench_ref${TAG}.json 2> gpurun_out/r2/bench_ref${TAG}.err; echo "rc=$?" >> gpurun_out/r2/bench_ref${TAG}.err
fi
