cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_halo -c 1 -o gpurun_out/prof_c1b python tools/gemm_probe.py --only-conv1 > gpurun_out/ncu_c1b.out 2>&1
ncu -i gpurun_out/prof_c1b.ncu-rep --page raw --csv > gpurun_out/prof_c1b_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_c1b.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_c1b_src.csv 2>/dev/null
