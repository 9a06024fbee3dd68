cd $GRAFT_REPO_ROOT
cat > gpurun_out/pp.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1408_5093_b200 as cb
cl = torch.channels_last
x = torch.relu(torch.randn(256, 96, 55, 55, device="cuda") - 0.3).to(torch.bfloat16).contiguous(memory_format=cl)
y, m = cb.pool_forward(x, "max", 3, 2, mask_dtype=torch.uint8)
dy = torch.randn_like(y)
dx = cb.pool_relu_backward(y, dy, m, tuple(x.shape), (3, 3), (2, 2), (0, 0))
torch.cuda.synchronize()
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k3s2 -o gpurun_out/prof_pool python gpurun_out/pp.py > gpurun_out/ncu_pool.out 2>&1
ncu -i gpurun_out/prof_pool.ncu-rep --page raw --csv > gpurun_out/prof_pool_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_pool.ncu-rep --page details --csv > gpurun_out/prof_pool_details.csv 2>/dev/null
tail -3 gpurun_out/ncu_pool.out
