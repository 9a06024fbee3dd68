"""Per-kernel device time of one CaffeNet training step (run on the B200 box).

Replays the CUDA-graph-captured step under torch.profiler (CUPTI kernel records, warm caches, the
real launch sequence) and prints, per kernel name and launch position, the mean device time per
step -- the breakdown that the ncu launch list gives cold and serialised.

    python tools/step_profile.py [--steps 10] [--json out.json]
"""
import argparse
import collections
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1408_5093_b200 import nets  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--json", default=None)
    ap.add_argument("--math", default="bf16", choices=["bf16", "tf32"])
    args = ap.parse_args()
    dev = torch.device("cuda")
    # CAFFE_TUNE="key=value,..." : library tuning knobs (caffe_set_tuning) for A/B runs
    from paper_1408_5093_b200 import _abi
    for kv in filter(None, os.environ.get("CAFFE_TUNE", "").split(",")):
        k, v = kv.split("=")
        _abi.call("caffe_set_tuning", int(k), int(v))
    net = nets.Net(nets.CAFFENET, args.batch, nets.CAFFENET_INPUT, dev, math=args.math, seed=0,
                   input_i8=args.math == "bf16")
    import synth
    net.a[0].copy_(torch.from_numpy(synth.int_pixels((args.batch,) + tuple(nets.CAFFENET_INPUT), 1000))
                   .to(net.a[0].dtype))
    net.labels.copy_(torch.from_numpy(synth.labels(args.batch, 1000, 1000)))
    for _ in range(3):
        net.step()
    torch.cuda.synchronize()
    graph = net.capture(overlap_update=os.environ.get("OVERLAP", "0") == "1")
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            graph.replay()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    per_step = len(evs) // args.steps
    seq = collections.OrderedDict()
    for i, e in enumerate(evs[: per_step * args.steps]):
        pos = i % per_step
        key = (pos, e.name.split("(")[0][:90])
        seq.setdefault(key, []).append(e.time_range.end - e.time_range.start)
    rows = [(pos, name, sum(v) / len(v)) for (pos, name), v in seq.items()]
    total = sum(r[2] for r in rows)
    by_name = collections.defaultdict(float)
    for _, name, us in rows:
        by_name[name] += us
    print(f"kernels per step: {per_step}; summed kernel time per step: {total:.1f} us")
    for pos, name, us in rows:
        print(f"{pos:4d} {us:9.1f} us  {name}")
    if os.environ.get("TIMELINE") == "1":
        # last profiled step: start / end relative to its first kernel, and the stream
        last = evs[per_step * (args.steps - 1): per_step * args.steps]
        t0 = min(e.time_range.start for e in last)
        print("--- timeline of the last step (us from its first kernel)")
        for e in sorted(last, key=lambda e: e.time_range.start):
            print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f}  s{getattr(e, 'device_resource_id', '?')}  {e.name.split('(')[0][:70]}")
    print("--- by kernel name")
    for name, us in sorted(by_name.items(), key=lambda kv: -kv[1]):
        print(f"{us:9.1f} us  {100 * us / total:5.1f}%  {name}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump({"per_step_us": total, "launches": [{"pos": p, "name": n, "us": u} for p, n, u in rows],
                       "by_name_us": by_name}, f, indent=1)


if __name__ == "__main__":
    main()
