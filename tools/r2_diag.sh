O=gpurun_out/r2diag
mkdir -p $O
for k in 4 2; do timeout 600 python tools/step_diag.py $k > $O/step_diag$k.txt 2>&1; done
for k in 4 2 3; do LAP_SETUP_TRACE=1 timeout 600 python tools/setup_trace.py $k > $O/setup_trace$k.txt 2>&1; done
