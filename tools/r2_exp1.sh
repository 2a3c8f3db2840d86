O=gpurun_out/r2exp1
mkdir -p $O
for k in 4 3 2; do
  timeout 300 python tools/exp_env.py $k default >> $O/exp.txt 2>&1
  LAP_SYMCHECK=search timeout 300 python tools/exp_env.py $k symsearch >> $O/exp.txt 2>&1
  LAP_SORT_ROWS=0 timeout 300 python tools/exp_env.py $k nosort >> $O/exp.txt 2>&1
done
