"""One eager CaffeNet training step bracketed by cudaProfilerStart/Stop (for ncu
--profile-from-start off): two warm-up steps, then the profiled step."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1408_5093_b200 import nets  # noqa: E402


def main():
    dev = torch.device("cuda")
    B = 256
    net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, dev, math="bf16", seed=0, input_i8=True)
    net.a[0].copy_(torch.from_numpy(synth.int_pixels((B,) + tuple(nets.CAFFENET_INPUT), 1000)).to(net.a[0].dtype))
    net.labels.copy_(torch.from_numpy(synth.labels(B, 1000, 1000)))
    for _ in range(2):
        net.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    net.step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
