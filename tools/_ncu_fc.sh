cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 6 -o gpurun_out/prof_fc6 python tools/gemm_probe.py --only-fc6w > gpurun_out/ncu_fc6.out 2>&1
ncu -i gpurun_out/prof_fc6.ncu-rep --page raw --csv > gpurun_out/prof_fc6_raw.csv 2>/dev/null
tail -3 gpurun_out/ncu_fc6.out
