"""CaffeNet conv2 data gradient (batch 256, 5x5, 2 groups of 48 -> 128 channels, BF16 channels-last)
with a filter row's taps in the MMA's N (CAFFE_TUNE_HALO_JN=1) against one MMA per tap (=0),
timed with CUDA events over graph-captured repeats (tools/gemm_probe.timeit).

    python tools/jn_probe.py [batch]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402
from gemm_probe import timeit  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    cl = torch.channels_last
    dev = torch.device("cuda")
    gf = 2.0 * n * 27 * 27 * 96 * 128 * 25 / 1e9
    x_shape = (n, 96, 27, 27)
    w = (torch.randn(256, 48, 5, 5, device=dev) * 0.05).to(torch.bfloat16)
    dy = torch.randn(n, 256, 27, 27, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
    dx = torch.empty(x_shape, device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)
    ws = cb.conv_workspace(x_shape, w.shape, 1, 2, 2, "bf16", 1, dev)
    res = {}
    for jn in (0, 1, 0, 1):
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_JN, jn)
        t = timeit(lambda: cb.conv_backward_data(dy, w, x_shape, 1, 2, 2, "bf16", out=dx, ws=ws))
        torch.cuda.synchronize()
        res[jn] = dx.float().clone()
        print(f"conv2 dgrad batch {n} jn={jn}: {t * 1e3:.1f} us ({gf / t:.0f} TFLOP/s algorithmic)", flush=True)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_JN, 1)
    d = (res[1] - res[0]).abs().max().item()
    r = (res[1] - res[0]).norm().item() / res[0].norm().item()
    print(f"jn vs per-tap: max|diff| {d:.3g}, rel-L2 {r:.3g}")


if __name__ == "__main__":
    main()
