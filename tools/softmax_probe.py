"""Softmax-with-loss at the CaffeNet shape (256 x 1000 FP32 scores, BF16 diff), CUDA events over
graph-captured repeats (tools/gemm_probe.timeit)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from gemm_probe import timeit  # noqa: E402

dev = torch.device("cuda")
s = torch.randn(256, 1000, device=dev) * 3
lab = torch.randint(0, 1000, (256,), device=dev, dtype=torch.int32)
loss = torch.zeros((), device=dev)
d = torch.empty(256, 1000, device=dev, dtype=torch.bfloat16)
t = timeit(lambda: cb.softmax_loss(s, lab, loss=loss, diff=d))
print(f"softmax loss 256x1000: {t * 1e3:.2f} us", flush=True)
