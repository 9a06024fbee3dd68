cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k 'regex:pack_s2d|maxpool|lrn_bwd|partial_reduce|sgd|bias_partial_nhwc8|wgrad_reduce' -o gpurun_out/prof_misc python tools/one_step.py > gpurun_out/ncu_misc.out 2>&1
ncu -i gpurun_out/prof_misc.ncu-rep --page raw --csv > gpurun_out/prof_misc_raw.csv 2>/dev/null
tail -3 gpurun_out/ncu_misc.out
