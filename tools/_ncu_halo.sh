cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_halo -c 4 -o gpurun_out/prof_halo python tools/gemm_probe.py --only-conv2 > gpurun_out/ncu_halo.out 2>&1
ncu -i gpurun_out/prof_halo.ncu-rep --page raw --csv > gpurun_out/prof_halo_raw.csv 2>/dev/null
tail -2 gpurun_out/ncu_halo.out
