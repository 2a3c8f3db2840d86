mkdir -p gpurun_out/r2
CFGS="4 3" bash tools/call_trace.sh
SCALE=26 TAG=_s26b bash tools/call_cfg5.sh
