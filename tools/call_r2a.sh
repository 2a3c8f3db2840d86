mkdir -p gpurun_out/r2
nvidia-smi > gpurun_out/r2/nvsmi.txt 2>&1
./tools/micro/gather 6534.5 > gpurun_out/r2/gather_micro.txt 2>&1
timeout 600 python tools/prof_solve.py 4 > gpurun_out/r2/levels_p4.txt 2>&1
timeout 600 python tools/prof_solve.py 3 > gpurun_out/r2/levels_p3.txt 2>&1
