"""Per-GPU time of the data-parallel CaffeNet step (bucketed all-reduce hooks, update after
finish), run as a one-rank NCCL group on one B200: the W > 1 code path minus the communication.
Compares the weight gradients on their own stream with the serial schedule."""
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1408_5093_b200 import nets  # noqa: E402
from paper_1408_5093_b200.dp import GradAllReduce  # noqa: E402


def main():
    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29544", rank=0, world_size=1)
    B = 256
    net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, torch.device("cuda"), math="bf16", seed=0, input_i8=True)
    net.a[0].copy_(torch.from_numpy(synth.int_pixels((B, 3, 227, 227), 1000)).to(net.a[0].dtype))
    net.labels.copy_(torch.from_numpy(synth.labels(B, 1000, 1000)))
    ar = GradAllReduce(net.grads, net.segments, 1)
    res = {}
    for _ in range(3):
        for side in (True, False):
            net.wgrad_side = side
            for _ in range(3):
                net.step(ar)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10):
                net.step(ar)
            b.record()
            torch.cuda.synchronize()
            res.setdefault(side, []).append(a.elapsed_time(b) / 10)
    for side, v in res.items():
        print(f"wgrad_side={side}: median {statistics.median(v):.4f} ms/step (eager, one-rank NCCL)  {v}")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
