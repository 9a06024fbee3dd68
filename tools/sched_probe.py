"""A/B timing of CUDA-graph-replayed CaffeNet steps under library tuning knobs and net schedule
options (run on the B200 box).

    python tools/sched_probe.py "flush=1073741824" "flush=6" "flush=6,blocks=2" "tune11=0"

Each argument is one configuration: comma-separated key=value with keys flush (Net.sgd_flush_layer),
blocks (Net.side_sgd_blocks), wside (Net.wgrad_side) and tuneK (caffe_set_tuning(K, value)).  Configurations are timed
round-robin (3 rounds x 20 replays) and the median ms/step of each is printed.
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1408_5093_b200 import _abi, nets  # noqa: E402


def parse(cfg):
    out = {}
    for kv in filter(None, cfg.split(",")):
        k, v = kv.split("=")
        out[k] = int(v)
    return out


def main():
    cfgs = sys.argv[1:] or [""]
    B = 256
    dev = torch.device("cuda")
    net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, dev, math="bf16", seed=0)
    net.a[0].copy_(torch.from_numpy(synth.int_pixels((B,) + tuple(nets.CAFFENET_INPUT), 1000)).to(torch.bfloat16))
    net.labels.copy_(torch.from_numpy(synth.labels(B, 1000, 1000)))
    graphs = []
    for c in cfgs:
        p = parse(c)
        for k, v in p.items():
            if k.startswith("tune"):
                _abi.call("caffe_set_tuning", int(k[4:]), v)
        net.sgd_flush_layer = p.get("flush", None)
        net.side_sgd_blocks = p.get("blocks", 1)
        net.side_sgd_threads = p.get("threads", 256)
        net.wgrad_side = bool(p.get("wside", 1))
        net.skip_update = bool(p.get("nosgd", 0))   # probe only: no parameter update (SGD cost)
        net.fuse_ip_sgd = bool(p.get("fuse", 0))
        net.fuse_ip_relu = bool(p.get("iprelu", 1))
        net.main_priority = -p.get("pmain", 2)
        net.wgrad_priority = -p.get("pwgrad", 1)
        net.sgd_priority = -p.get("psgd", 0)
        net._side = None
        net._wside = None
        for _ in range(2):
            net.step()
        torch.cuda.synchronize()
        graphs.append(net.capture())
        for k, v in p.items():   # restore library defaults (tuning is process-wide)
            if k.startswith("tune"):
                _abi.call("caffe_set_tuning", int(k[4:]), 1 if int(k[4:]) in (5, 10, 11) else (1 if int(k[4:]) == 14 else 0))
    res = {c: [] for c in cfgs}
    rounds = int(os.environ.get("ROUNDS", "3"))
    for _ in range(rounds):
        for c, g in zip(cfgs, graphs):
            for _ in range(3):
                g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(20):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            res[c].append(a.elapsed_time(b) / 20)
    for c in cfgs:
        print(f"{c:40s} median {statistics.median(res[c]):.4f}  min {min(res[c]):.4f} ms/step  "
              f"{['%.4f' % x for x in res[c]]}")


if __name__ == "__main__":
    main()
