"""conv1 / conv2 forward and conv2 data-gradient timing under library tuning knobs (run on the B200
box): python tools/conv1_probe.py "11=1" "11=0" "12=1"  (key=value pairs of caffe_set_tuning).
(This round's store probes -- the epilogue without global stores: conv1 forward 81 -> 54 us -- used
a since-removed debug knob.)"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402
from gemm_probe import timeit  # noqa: E402


# library defaults of the knobs the probe sets (restored after each configuration)
DEFAULTS = {5: 1, 10: 1, 11: 1, 12: 0, 18: 1, 22: 1}


def main():
    dev = torch.device("cuda")
    B = 256
    x = torch.randint(-128, 128, (B, 3, 227, 227), device=dev).float().to(torch.bfloat16).contiguous(
        memory_format=torch.channels_last)
    w = (torch.randn(96, 3, 11, 11, device=dev) * 0.01).to(torch.bfloat16)
    b = torch.zeros(96, device=dev)
    y = torch.empty((B, 96, 55, 55), device=dev, dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
    ws = cb.conv_bottom_workspace(x.shape, w.shape, 4, 0, 1, "bf16", dev)
    cb.conv_pack_bottom(x, w, 4, 0, 1, "bf16", ws=ws)
    # conv2 shapes
    x2 = torch.randn(B, 96, 27, 27, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    w2 = (torch.randn(256, 48, 5, 5, device=dev) * 0.01).to(torch.bfloat16)
    b2 = torch.zeros(256, device=dev)
    y2 = torch.empty((B, 256, 27, 27), device=dev, dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
    # conv2 data gradient (N = 48 per group)
    dy2 = torch.randn(B, 256, 27, 27, device=dev).to(torch.bfloat16).contiguous(memory_format=torch.channels_last)
    dx2 = torch.empty((B, 96, 27, 27), device=dev, dtype=torch.bfloat16).contiguous(memory_format=torch.channels_last)
    for cfg in sys.argv[1:] or ["11=1", "11=0", "12=1"]:
        kv = [tuple(map(int, s.split("="))) for s in cfg.split(",")]
        for k, v in kv:
            _abi.call("caffe_set_tuning", k, v)
        t1 = timeit(lambda: cb.conv_forward(x, w, b, 4, 0, 1, "bf16", relu=True, out=y, ws=ws, prepacked=True))
        t2 = timeit(lambda: cb.conv_forward(x2, w2, b2, 1, 2, 2, "bf16", relu=True, out=y2))
        t3 = timeit(lambda: cb.conv_backward_data(dy2, w2, x2.shape, 1, 2, 2, "bf16", out=dx2))
        print(f"{cfg:20s} conv1 fwd {t1 * 1e3:7.1f} us   conv2 fwd {t2 * 1e3:7.1f} us   conv2 dgrad {t3 * 1e3:7.1f} us",
              flush=True)
        for k, v in kv:
            _abi.call("caffe_set_tuning", k, DEFAULTS.get(k, 0))


if __name__ == "__main__":
    main()
