"""Step time (graph replay, CaffeNet batch 256, one B200) under schedule variants of nets.Net:
    python tools/sched_sweep.py "wgrad_max_ctas=0" "wgrad_max_ctas=96" ...
Each argument is a comma-separated list of Net attribute assignments; "tuneK=V" entries set library
tuning knob K (caffe_set_tuning) instead, and each such configuration runs in a fresh process."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1408_5093_b200 import nets  # noqa: E402


def run(assign):
    if ("tune" in assign or "cls." in assign) and os.environ.get("SCHED_SWEEP_CHILD") != "1":
        import subprocess
        out = subprocess.run([sys.executable, os.path.abspath(__file__), assign], capture_output=True, text=True,
                             env=dict(os.environ, SCHED_SWEEP_CHILD="1", REPS="1"), timeout=600).stdout
        return float(out.strip().splitlines()[-1].split()[-4]) / 1e3
    from paper_1408_5093_b200 import _abi
    dev = torch.device("cuda")
    for kv in filter(None, assign.split(",")):   # "cls.X=V": a Net class attribute read at construction
        k, v = kv.split("=")
        if k.startswith("cls."):
            setattr(nets.Net, k[4:], type(getattr(nets.Net, k[4:]))(eval(v)))
    net = nets.Net(nets.CAFFENET, 256, nets.CAFFENET_INPUT, dev, math="bf16", seed=0, input_i8=True)
    for kv in filter(None, assign.split(",")):
        k, v = kv.split("=")
        if k.startswith("cls."):
            continue
        if k.startswith("tune"):
            _abi.call("caffe_set_tuning", int(k[4:]), int(eval(v)))
        else:
            cur = getattr(net, k)
            setattr(net, k, eval(v) if cur is None else type(cur)(eval(v)))
    net.a[0].copy_(torch.from_numpy(synth.int_pixels((256, 3, 227, 227), 1000)).to(net.a[0].dtype))
    net.labels.copy_(torch.from_numpy(synth.labels(256, 1000, 1000)))
    for _ in range(3):
        net.step()
    torch.cuda.synchronize()
    g = net.capture()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 10)
    t = sorted(ts)[2]
    del net, g
    torch.cuda.empty_cache()
    return t


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["wgrad_max_ctas=0"]
    reps = int(os.environ.get("REPS", "2"))
    res = {c: [] for c in cfgs}
    for rep in range(reps):
        for c in cfgs:
            res[c].append(run(c) * 1e3)
            print(f"{c:40s} {res[c][-1]:8.1f} us/step", flush=True)
    for c in cfgs:
        v = sorted(res[c])
        print(f"median {c:33s} {v[len(v) // 2]:8.1f} us/step  (min {v[0]:.1f})", flush=True)
