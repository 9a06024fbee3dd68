"""conv1 weight gradient (CaffeNet, batch 256: 148 pixel splits) + its split reduction, with the
wide (16/32 threads per output) reduction on and off; CUDA-event time of the pair.
    python tools/reduce_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402
from gemm_probe import timeit  # noqa: E402


def main():
    dev = torch.device("cuda")
    cl = torch.channels_last
    x = torch.randint(-128, 128, (256, 3, 227, 227), device=dev).to(torch.int8).contiguous(memory_format=cl)
    w = (torch.randn(96, 3, 11, 11, device=dev) * 0.01).to(torch.bfloat16)
    dy = torch.randn(256, 96, 55, 55, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
    dw, db = torch.empty(96, 3, 11, 11, device=dev), torch.empty(96, device=dev)
    ws = cb.conv_bottom_workspace(x.shape, w.shape, 4, 0, 1, "bf16", dev)
    cb.conv_pack_bottom(x, w, 4, 0, 1, "bf16", ws=ws)
    res = {}
    for wide in (0, 1, 0, 1):
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_REDUCE_WIDE, wide)
        t = timeit(lambda: cb.conv_backward_weight(x, dy, w.shape, 4, 0, 1, "bf16", beta=0.0, dw=dw, db=db, ws=ws,
                                                   prepacked=True))
        res.setdefault(wide, []).append(t * 1e3)
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_REDUCE_WIDE, 1)
    print("conv1 wgrad + reduce us: " + " ".join(f"wide={k}: {v}" for k, v in res.items()))


if __name__ == "__main__":
    main()
