"""The 13x13 CaffeNet passes (conv3-5 forward and data gradient, batch 256, BF16 channels-last)
under each tile form: per-tap im2col tiles, stacked halo tiles (one or two accumulators per CTA),
timed with CUDA events over graph-captured repeats (tools/gemm_probe.timeit).

    python tools/conv13_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402
from gemm_probe import timeit  # noqa: E402

LAYERS = [("conv3", 256, 384, 1, 76.55), ("conv4", 384, 384, 2, 57.42), ("conv5", 384, 256, 2, 38.28)]
MODES = [("im2col", 0), ("stacked auto", 1), ("stacked force", 2), ("stacked 2acc", 3), ("stacked bn<=128", 4)]


def main():
    cl = torch.channels_last
    dev = torch.device("cuda")
    for name, C, O, g, gf in LAYERS:
        x = torch.randn(256, C, 13, 13, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
        w = (torch.randn(O, C // g, 3, 3, device=dev) * 0.05).to(torch.bfloat16)
        b = torch.zeros(O, device=dev)
        y = torch.empty(256, O, 13, 13, device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)
        dy = torch.randn(256, O, 13, 13, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
        dx = torch.empty_like(x)
        wsf = cb.conv_workspace(x.shape, w.shape, 1, 1, g, "bf16", 0, dev)
        wsd = cb.conv_workspace(x.shape, w.shape, 1, 1, g, "bf16", 1, dev)
        line = [f"{name}:"]
        ref_y = ref_dx = None
        for mname, mode in MODES:
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_STACKED, mode)
            tf = timeit(lambda: cb.conv_forward(x, w, b, 1, 1, g, "bf16", relu=True, out=y, ws=wsf))
            td = timeit(lambda: cb.conv_backward_data(dy, w, x.shape, 1, 1, g, "bf16", out=dx, ws=wsd))
            torch.cuda.synchronize()
            if ref_y is None:
                ref_y, ref_dx = y.float().clone(), dx.float().clone()
            ey = float((y.float() - ref_y).abs().max())
            ed = float((dx.float() - ref_dx).abs().max())
            line.append(f"{mname} fwd {tf * 1e3:.1f} us ({gf / tf:.0f} TF) dgrad {td * 1e3:.1f} us "
                        f"({gf / td:.0f} TF) [max|diff| {ey:.2g}/{ed:.2g}]")
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_STACKED, 1)
        print("\n  ".join(line), flush=True)


if __name__ == "__main__":
    main()
