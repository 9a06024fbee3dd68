import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import paper_1408_5093_b200 as cb
from paper_1408_5093_b200 import _abi
from gemm_probe import timeit
dev = torch.device("cuda")
for name, K, O in [("fc6", 9216, 4096), ("fc7", 4096, 4096), ("fc8", 4096, 1000)]:
    x = torch.randn(256, K, device=dev).to(torch.bfloat16)
    w = (torch.randn(O, K, device=dev) * 0.005).to(torch.bfloat16)
    b = torch.zeros(O, device=dev)
    y = torch.empty(256, O, device=dev, dtype=torch.bfloat16)
    dy = torch.randn(256, O, device=dev).to(torch.bfloat16)
    dx = torch.empty(256, K, device=dev, dtype=torch.bfloat16)
    line = [name]
    for cap in (0, 16, 8, 4, 2):
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_IP_MAX_SPLITS, cap)
        tf = timeit(lambda: cb.ip_forward(x, w, b, "bf16", relu=True, out=y))
        td = timeit(lambda: cb.ip_backward_data(dy, w, x.shape, "bf16", out=dx))
        line.append(f"cap {cap}: fwd {tf*1e3:.1f} dgrad {td*1e3:.1f}")
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_IP_MAX_SPLITS, 0)
    print(" | ".join(line), flush=True)
