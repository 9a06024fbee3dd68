import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import paper_1408_5093_b200 as cb
from paper_1408_5093_b200 import _abi
from gemm_probe import timeit
dev = torch.device("cuda")
for O, K in [(1000, 4096), (4096, 4096)]:
    x = torch.randn(256, K, device=dev).to(torch.bfloat16)
    dy = torch.randn(256, O, device=dev).to(torch.bfloat16)
    dw = torch.zeros(O, K, device=dev); db = torch.zeros(O, device=dev)
    line = [f"O={O}"]
    for r in (64, 32, 16, 8):
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_BIAS_SPLIT_ROWS, r)
        t1 = timeit(lambda: cb.ip_backward_weight(x, dy, (O, K), "bf16", dw=dw, db=db))
        t0 = timeit(lambda: cb.ip_backward_weight(x, dy, (O, K), "bf16", dw=dw, bias=False))
        line.append(f"rows {r}: bias {1e3*(t1-t0):.1f} us")
    print(" | ".join(line), flush=True)
_abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_BIAS_SPLIT_ROWS, 64)
