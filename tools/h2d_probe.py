"""Host->device bandwidth of the bench's per-step input (pinned int8 batch, 39.6 MB) alone and beside
the captured training step (run on the B200 box)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1408_5093_b200 import nets  # noqa: E402


def main():
    dev = torch.device("cuda")
    B = 256
    hX = torch.from_numpy(synth.int_pixels((B, 3, 227, 227), 1000)).to(torch.int8) \
        .contiguous(memory_format=torch.channels_last).pin_memory()
    d = torch.empty_like(hX, device=dev)
    for _ in range(3):
        d.copy_(hX, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        d.copy_(hX, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"H2D alone: {ms:.3f} ms per 39.6 MB batch = {hX.numel() / ms / 1e6:.1f} GB/s")
    net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, dev, math="bf16", seed=0, input_i8=True)
    net.a[0].copy_(hX)
    net.labels.copy_(torch.from_numpy(synth.labels(B, 1000, 1000)))
    for _ in range(3):
        net.step()
    g = net.capture()
    cs = torch.cuda.Stream()
    torch.cuda.synchronize()
    for K in (20, 100):
        e0.record()
        for _ in range(K):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        tg = e0.elapsed_time(e1) / K
        # replays with the next batch's copy running beside each (copy stream)
        e0.record()
        for _ in range(K):
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                d.copy_(hX, non_blocking=True)
            g.replay()
        torch.cuda.current_stream().wait_stream(cs)
        e1.record()
        torch.cuda.synchronize()
        tc = e0.elapsed_time(e1) / K
        print(f"K={K}: replay {tg:.3f} ms/step, replay + concurrent H2D {tc:.3f} ms/step")


if __name__ == "__main__":
    main()
