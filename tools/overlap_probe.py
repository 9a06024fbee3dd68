"""Does a side-stream SGD update overlap the main stream's backward kernels?  Eager and graph
timelines of Net.step(overlap_update=True) (CUPTI kernel start/end, stream id)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1408_5093_b200 import nets  # noqa: E402


def timeline(fn, label):
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    end = max(e.time_range.end for e in evs) - t0
    print(f"== {label}: span {end:.1f} us")
    for e in evs:
        if "sgd" in e.name or "maxpool_bwd" in e.name or "tc_" in e.name:
            print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {getattr(e, 'device_resource_id', '?')} "
                  f"{e.name.split('(')[0][:50]}")


def main():
    B = 256
    net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, torch.device("cuda"), math="bf16", seed=0)
    net.a[0].copy_(torch.from_numpy(synth.int_pixels((B,) + tuple(nets.CAFFENET_INPUT), 1000)).to(torch.bfloat16))
    net.labels.copy_(torch.from_numpy(synth.labels(B, 1000, 1000)))
    for _ in range(3):
        net.step(overlap_update=True)
    timeline(lambda: net.step(overlap_update=True), "eager overlap")
    timeline(lambda: net.step(overlap_update=False), "eager serial")
    # graph-replayed step times, overlap on / off
    for ov, bps in ((False, 1), (True, 1), (True, 2), (True, 4)):
        net.side_sgd_blocks = bps
        g = net.capture(overlap_update=ov)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            g.replay()
        b.record()
        b.synchronize()
        print(f"graph overlap={ov} sgd_blocks_per_sm={bps}: {a.elapsed_time(b) / 20 * 1000:.1f} us/step")


if __name__ == "__main__":
    main()
