# Round profile capture (run on the GPU box through gpurun): the launch list of one training step
# and a full-set capture of its tensor-core GEMM launches.
cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file gpurun_out/launches_step.csv python tools/one_step.py > gpurun_out/ncu_list.out 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off -k 'regex:tc_gemm|tc_halo' \
  -o gpurun_out/prof_step_gemm python tools/one_step.py > gpurun_out/ncu_full.out 2>&1
ncu -i gpurun_out/prof_step_gemm.ncu-rep --page raw --csv > gpurun_out/prof_step_gemm_raw.csv 2>/dev/null
tail -n 2 gpurun_out/ncu_list.out gpurun_out/ncu_full.out
