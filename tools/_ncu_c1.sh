cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_halo -c 3 -o gpurun_out/prof_c1 python tools/gemm_probe.py --only-conv1 > gpurun_out/ncu_c1.out 2>&1
ncu -i gpurun_out/prof_c1.ncu-rep --page raw --csv > gpurun_out/prof_c1_raw.csv 2>/dev/null
for r in 0 1; do timeout 100 python tools/gemm_probe.py --rows $r 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('rows', $r, d['conv1']['fwd_us'], d['conv2']['fwd_us'], d['conv2']['dgrad_us'])"; done
