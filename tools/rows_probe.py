import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import torch
import paper_1408_5093_b200 as cb
from paper_1408_5093_b200 import _abi
from gemm_probe import timeit
dev = torch.device("cuda")
x = torch.randn(256, 256, 6, 6, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
w = (torch.randn(4096, 9216, device=dev) * 0.005).to(torch.bfloat16)
y = torch.empty(256, 4096, device=dev, dtype=torch.bfloat16)
xr = x.contiguous().view(256, -1)
t0 = timeit(lambda: cb.ip_forward(xr, w, None, "bf16", out=y))
for v in (0, 1, 0, 1):
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_ROWS_CB, v)
    t = timeit(lambda: cb.ip_forward(x, w, None, "bf16", out=y))
    print(f"fc6 fwd from NHWC rows_cb={v}: {t*1e3:.1f} us (from rows {t0*1e3:.1f} us: staging {1e3*(t-t0):.1f} us)", flush=True)
_abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_ROWS_CB, 1)
