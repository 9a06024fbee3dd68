"""Where does the end-to-end step (bench.py's e2e leg) lose time against the device-only step?  Two
captured step graphs reading two input blobs, as in bench.py, timed over K replays with (a) the
bench's input pipeline: H2D of the next batch into the other blob on a copy stream + the labels
H2D and the loss D2H on the compute stream, (b) the big copy only, (c) the small copies only,
(d) replays only (run on the B200 box)."""
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_1408_5093_b200 import nets  # noqa: E402


def main():
    B, K = 256, 20
    dev = torch.device("cuda")
    net = nets.Net(nets.CAFFENET, B, nets.CAFFENET_INPUT, dev, math="bf16", seed=0, input_i8=True)
    X = synth.int_pixels((B, 3, 227, 227), 1000)
    net.a[0].copy_(torch.from_numpy(X).to(net.a[0].dtype))
    net.labels.copy_(torch.from_numpy(synth.labels(B, 1000, 1000)))
    for _ in range(3):
        net.step()
    torch.cuda.synchronize()
    dstage = [net.a[0], torch.empty_like(net.a[0])]
    graphs = [net.capture()]
    a0 = net.a[0]
    net.a[0] = dstage[1]
    graphs.append(net.capture())
    net.a[0] = a0
    stream = torch.cuda.current_stream()
    cl = torch.channels_last
    hX = torch.from_numpy(X).to(net.a[0].dtype).contiguous(memory_format=cl).pin_memory()
    hL = torch.from_numpy(synth.labels(B, 1000, 1000)).pin_memory()
    hloss = torch.empty((), dtype=torch.float32).pin_memory()
    cs = torch.cuda.Stream()
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]

    dX = torch.empty_like(net.a[0])
    dX.copy_(hX)

    def run(h2d, small, src=None):
        torch.cuda.synchronize()
        time.sleep(0.5)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)

        def prefetch(i):
            k = i % 2
            cs.wait_stream(stream) if i < 2 else cs.wait_event(consumed[k])
            with torch.cuda.stream(cs):
                dstage[k].copy_(hX if src is None else src, non_blocking=True)
                copied[k].record(cs)
        if h2d:
            prefetch(0)
        for i in range(K):
            k = i % 2
            if h2d:
                if i + 1 < K:
                    prefetch(i + 1)
                stream.wait_event(copied[k])
            if small:
                net.labels.copy_(hL, non_blocking=True)
            graphs[k].replay()
            consumed[k].record(stream)
            if small:
                hloss.copy_(net.loss, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    cfgs = [("bench", (1, 1)), ("h2d_only", (1, 0)), ("d2d_only", (1, 0, dX)), ("small_only", (0, 1)),
            ("replay_only", (0, 0))]
    res = {n: [] for n, _ in cfgs}
    for _ in range(4):
        for name, cfg in cfgs:
            res[name].append(run(*cfg))
    for name, _ in cfgs:
        print(f"{name:12s} median {statistics.median(res[name]):.4f} ms/step  {['%.3f' % x for x in res[name]]}",
              flush=True)


if __name__ == "__main__":
    main()
