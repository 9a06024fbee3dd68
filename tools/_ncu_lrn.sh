# ncu --set full of the LRN / pool kernels of one eager CaffeNet step; details page as CSV
cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --profile-from-start off -k 'regex:lrn|pool' -o gpurun_out/prof_lrn python tools/one_step.py > gpurun_out/ncu_lrn.out 2>&1
ncu -i gpurun_out/prof_lrn.ncu-rep --page details --csv > gpurun_out/prof_lrn_details.csv 2>/dev/null
ncu -i gpurun_out/prof_lrn.ncu-rep --page raw --csv > gpurun_out/prof_lrn_raw.csv 2>/dev/null
tail -2 gpurun_out/ncu_lrn.out
