"""CaffeNet conv1 forward (batch 256, int8-exact pixels packed by space-to-depth, BF16 channels-last
output, bias + ReLU) with one shared window per CTA's two row blocks (CAFFE_TUNE_HALO_MERGE=1) or one
window per tile (=0), timed with CUDA events over graph-captured repeats (tools/gemm_probe.timeit).

    python tools/merge_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402
from gemm_probe import timeit  # noqa: E402


def main():
    cl = torch.channels_last
    dev = torch.device("cuda")
    n = 256
    gf = 2.0 * n * 55 * 55 * 96 * 3 * 121 / 1e9
    x = torch.randint(-128, 128, (n, 3, 227, 227), device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
    w = (torch.randn(96, 3, 11, 11, device=dev) * 0.01).to(torch.bfloat16)
    b = torch.zeros(96, device=dev)
    y = torch.empty(n, 96, 55, 55, device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)
    ws = cb.conv_workspace(x.shape, w.shape, 4, 0, 1, "bf16", 0, dev)
    res = {}
    for m in (0, 1, 0, 1):
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_MERGE, m)
        t = timeit(lambda: cb.conv_forward(x, w, b, 4, 0, 1, "bf16", relu=True, out=y, ws=ws))
        torch.cuda.synchronize()
        res[m] = y.float().clone()
        print(f"conv1 forward (incl. s2d pack) merge={m}: {t * 1e3:.1f} us ({gf / t:.0f} TFLOP/s)", flush=True)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_MERGE, 0)
    print("bit-identical:", bool(torch.equal(res[0], res[1])))


if __name__ == "__main__":
    main()
