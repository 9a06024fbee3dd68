"""fc8 forward (256 x 4096 -> 1000, BF16) under CAFFE_TUNE_IP_FWD_SMALL_BN (0 = general N tile, 64,
128): GEMM + split-K reduce, CUDA events over graph-captured repeats (tools/gemm_probe.timeit)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402
from gemm_probe import timeit  # noqa: E402

dev = torch.device("cuda")
x = torch.randn(256, 4096, device=dev).to(torch.bfloat16)
w = (torch.randn(1000, 4096, device=dev) * 0.01).to(torch.bfloat16)
b = torch.zeros(1000, device=dev)
y = torch.empty(256, 1000, device=dev, dtype=torch.float32)
ref = None
for v in (0, 64, 128, 0, 64, 128):
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_IP_FWD_SMALL_BN, v)
    t = timeit(lambda: cb.ip_forward(x, w, b, "bf16", out=y))
    torch.cuda.synchronize()
    if ref is None:
        ref = y.clone()
    print(f"fc8 fwd small_bn={v}: {t * 1e3:.1f} us  max|diff| {float((y - ref).abs().max()):.2e}", flush=True)
_abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_IP_FWD_SMALL_BN, 0)
