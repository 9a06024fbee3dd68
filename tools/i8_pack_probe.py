"""The int8 image pack of CaffeNet's first layer (batch 256, 3x227x227 -> space-to-depth 57x57x48 BF16):
one-thread-per-packed-pixel kernel (CAFFE_TUNE_I8_ROWS=1) against the 12-byte segment kernel (=0), CUDA events over
graph-captured repeats (tools/gemm_probe.timeit).

    python tools/i8_pack_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402
from gemm_probe import timeit  # noqa: E402


def main():
    dev = torch.device("cuda")
    x = torch.randint(-128, 128, (256, 3, 227, 227), device=dev, dtype=torch.int8).contiguous(memory_format=torch.channels_last)
    w = (torch.randn(96, 3, 11, 11, device=dev) * 0.01).to(torch.bfloat16)
    ws = cb.conv_bottom_workspace(x.shape, w.shape, 4, 0, 1, "bf16", dev)
    mb = (x.numel() + 256 * 57 * 57 * 48 * 2) / 1e6
    res = {}
    for r in (0, 1, 2, 0, 1, 2):
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_I8_ROWS, r)
        t = timeit(lambda: cb.conv_pack_bottom(x, w, 4, 0, 1, "bf16", ws=ws))
        torch.cuda.synchronize()
        res[r] = ws.clone()
        print(f"i8 pack rows={r}: {t * 1e3:.1f} us ({mb / t / 1e3:.2f} TB/s algorithmic)", flush=True)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_I8_ROWS, 1)
    print("workspace bit-identical:", bool(torch.equal(res[0], res[1])))


if __name__ == "__main__":
    main()
