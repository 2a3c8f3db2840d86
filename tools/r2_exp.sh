# generic: GPU tests subset (PYTEST_K) + exp_env on configs (CFGS) with env settings (ENVS, ';'-separated)
O=gpurun_out/${OUT:-r2exp}
mkdir -p $O
if [ -n "$PYTEST_K" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$PYTEST_K" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
fi
IFS=';' read -ra EV <<< "${ENVS:-default=1}"
for k in ${CFGS:-4 3 2}; do
  for e in "${EV[@]}"; do
    env $e timeout 300 python tools/exp_env.py $k "$e" >> $O/exp.txt 2>> $O/exp.err
  done
done
