"""TF32 conv weight-gradient timings (CaffeNet conv2-5 shapes, batch 256, FP32 channels-last blobs)
for each CAFFE_TUNE_WGRAD_MACC setting, and the TF32 training step.
    python tools/tf32_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402
from gemm_probe import timeit  # noqa: E402

LAYERS = [("conv2", 96, 27, 256, 5, 2, 2, 114.66), ("conv3", 256, 13, 384, 3, 1, 1, 76.55),
          ("conv4", 384, 13, 384, 3, 1, 2, 57.42), ("conv5", 384, 13, 256, 3, 1, 2, 38.28)]


def main():
    dev = torch.device("cuda")
    cl = torch.channels_last
    for name, C, H, O, k, p, g, gf in LAYERS:
        x = torch.randn(256, C, H, H, device=dev).contiguous(memory_format=cl)
        dy = torch.randn(256, O, H, H, device=dev).contiguous(memory_format=cl)
        dw = torch.empty(O, C // g, k, k, device=dev)
        db = torch.empty(O, device=dev)
        line = [f"{name} TF32 wgrad:"]
        for m in (0, 1, 2, 3, 4):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_MACC, m)
            ws = cb.conv_workspace(x.shape, dw.shape, 1, p, g, "tf32", 2, dev)
            t = timeit(lambda: cb.conv_backward_weight(x, dy, dw.shape, 1, p, g, "tf32", beta=0.0, dw=dw, db=db, ws=ws))
            line.append(f"macc{m} {t * 1e3:.1f} us ({gf / t:.0f} TF)")
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_MACC, 0)
        wsf = cb.conv_workspace(x.shape, dw.shape, 1, p, g, "tf32", 0, dev)
        y = torch.empty(256, O, H, H, device=dev).contiguous(memory_format=cl)
        t = timeit(lambda: cb.conv_forward(x, dw, db, 1, p, g, "tf32", out=y, ws=wsf))
        line.append(f"| fwd {t * 1e3:.1f} us ({gf / t:.0f} TF)")
        print(" ".join(line), flush=True)


if __name__ == "__main__":
    main()
