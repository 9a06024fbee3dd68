# full ncu capture (with source) of the conv1 forward halo kernel, exported as raw + source CSV
cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_halo --launch-skip 2 -c 1 -o gpurun_out/prof_c1s python tools/gemm_probe.py --only-conv1 > gpurun_out/ncu_c1s.out 2>&1
ncu -i gpurun_out/prof_c1s.ncu-rep --page raw --csv > gpurun_out/prof_c1s_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_c1s.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_c1s_sass.csv 2>/dev/null
ncu -i gpurun_out/prof_c1s.ncu-rep --page details --csv > gpurun_out/prof_c1s_details.csv 2>/dev/null
