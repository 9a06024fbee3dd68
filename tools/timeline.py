"""Kernel timeline of one graph-replayed CaffeNet step (start/end in us, stream id) -- to check
which launches overlap (e.g. the side-stream SGD updates)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1408_5093_b200 import nets  # noqa: E402


def main():
    B = 256
    net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, torch.device("cuda"), math="bf16", seed=0, input_i8=True)
    from paper_1408_5093_b200 import _abi
    for kv in filter(None, os.environ.get("CAFFE_TUNE", "").split(",")):   # library knobs "key=value,..."
        k, v = kv.split("=")
        _abi.call("caffe_set_tuning", int(k), int(v))
    # NET_ATTRS="attr=value,...": Net attribute overrides (as tools/sched_sweep.py)
    for kv in filter(None, os.environ.get("NET_ATTRS", "").split(",")):
        k, v = kv.split("=")
        setattr(net, k, type(getattr(net, k))(eval(v)))
    net.a[0].copy_(torch.from_numpy(synth.int_pixels((B,) + tuple(nets.CAFFENET_INPUT), 1000)).to(net.a[0].dtype))
    net.labels.copy_(torch.from_numpy(synth.labels(B, 1000, 1000)))
    for _ in range(3):
        net.step()
    torch.cuda.synchronize()
    g = net.capture()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.replay()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    for e in evs:
        print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.end - e.time_range.start:7.1f} "
              f"{getattr(e, 'device_resource_id', '?')} {e.name.split('(')[0][:60]}")


if __name__ == "__main__":
    main()
