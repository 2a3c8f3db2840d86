# ncu --set full of the main setup kernels of one warm cfg-k setup (NVTX range setup2)
O=gpurun_out/r2ncu
mkdir -p $O
K=${CFG:-4}
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "setup2/" \
  -k regex:"${KREGEX:-k_cspmv_store|k_vote_round|k_gal_slot_emit|k_perm_sort_thread|k_affinity}" -c ${NK:-24} \
  -o $O/setup_cfg$K python tools/prof_setup.py $K > $O/ncu_setup_cfg$K.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "setup2/" --csv \
  --log-file $O/launches_setup_cfg$K.csv python tools/prof_setup.py $K > $O/ncu_launch_setup_cfg$K.log 2>&1
