"""Time the channels-last BF16 max-pool forward / ReLU-fused backward at CaffeNet's pool shapes
(batch 256, U8 masks) for a sweep of CAFFE_TUNE_POOL_STRIP_ROWS values (run on the B200 box).

    python tools/pool_probe.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a.record()
        fn()
        b.record()
        b.synchronize()
        tot += a.elapsed_time(b)
    return tot / reps * 1000


def main():
    cl = torch.channels_last
    for (C, H) in ((96, 55), (256, 27), (256, 13)):
        x = torch.relu(torch.randn(256, C, H, H, device="cuda") - 0.3).to(torch.bfloat16).contiguous(memory_format=cl)
        y, m = cb.pool_forward(x, "max", 3, 2, mask_dtype=torch.uint8)
        dy = torch.randn_like(y)
        fwd = timed(lambda: cb.pool_forward(x, "max", 3, 2, out=y, mask=m))
        byts = x.numel() * 2 + y.numel() * 3
        line = f"C={C} H={H}: fwd {fwd:6.1f} us ({byts / fwd / 1e3:5.0f} GB/s)  bwd"
        ref = None
        for rows in (0, 1, 2, 3, 4, 7, 14, 28):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_POOL_STRIP_ROWS, rows)
            dx = cb.pool_relu_backward(y, dy, m, tuple(x.shape), (3, 3), (2, 2), (0, 0))
            if ref is None:
                ref = dx.clone()
            assert torch.equal(dx, ref), rows
            t = timed(lambda: cb.pool_relu_backward(y, dy, m, tuple(x.shape), (3, 3), (2, 2), (0, 0)))
            line += f"  r{rows}:{t:5.1f}"
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_POOL_STRIP_ROWS, 0)
        bb = x.numel() * 2 + y.numel() * 5
        print(line + f"   (bwd bytes {bb / 1e6:.0f} MB)")


if __name__ == "__main__":
    main()
