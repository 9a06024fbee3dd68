"""CaffeNet conv weight gradients (batch 256, BF16 channels-last, halo-tiled) under each N tile
(CAFFE_TUNE_WGRAD_BN), timed with CUDA events over graph-captured repeats (tools/gemm_probe.timeit).

    python tools/wgrad_probe.py [layer ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402
from gemm_probe import timeit  # noqa: E402

# name, C, H, O, k, stride, pad, group
LAYERS = {"conv1": (3, 227, 96, 11, 4, 0, 1), "conv2": (96, 27, 256, 5, 1, 2, 2), "conv3": (256, 13, 384, 3, 1, 1, 1),
          "conv4": (384, 13, 384, 3, 1, 1, 2), "conv5": (384, 13, 256, 3, 1, 1, 2)}
BNS = [0, 1, 64, 96, 128, 192, 256]


def main():
    names = sys.argv[1:] or list(LAYERS)
    cl = torch.channels_last
    dev = torch.device("cuda")
    n = 256
    for name in names:
        C, H, O, k, s, p, g = LAYERS[name]
        OH = (H + 2 * p - k) // s + 1
        gf = 2.0 * n * OH * OH * O * (C // g) * k * k / 1e9
        x = torch.randn(n, C, H, H, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
        dy = torch.randn(n, O, OH, OH, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
        dw = torch.zeros(O, C // g, k, k, device=dev)
        db = torch.zeros(O, device=dev)
        ref = None
        line = [f"{name} wgrad ({gf:.1f} GFLOP):"]
        for bn in BNS:
            if bn > 1 and bn > O // g and bn != 64:
                continue
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_BN, bn)
            ws = cb.conv_workspace(x.shape, dw.shape, s, p, g, "bf16", 2, dev)
            t = timeit(lambda: cb.conv_backward_weight(x, dy, dw.shape, s, p, g, "bf16", dw=dw, db=db, ws=ws))
            torch.cuda.synchronize()
            if ref is None:
                ref = dw.clone()
            d = float((dw - ref).norm() / ref.norm())
            line.append(f"BN {({0: 'auto', 1: 'widest'}).get(bn, bn)}: {t * 1e3:.1f} us ({gf / t:.0f} TF) [rel {d:.1e}]")
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_BN, 0)
        print("\n  ".join(line), flush=True)


if __name__ == "__main__":
    main()
