"""Where does the end-to-end step lose time against the device-only step?  Times K graph-replayed
steps with (a) the bench's full input pipeline, (b) without the host->device copy, (c) without
the device copy into the input blob, (d) replays only (run on the B200 box)."""
import os
import sys

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
    g = net.capture()
    stream = torch.cuda.current_stream()
    cl = torch.channels_last
    hX = torch.from_numpy(X).to(net.a[0].dtype).contiguous(memory_format=cl).pin_memory()
    hL = torch.from_numpy(synth.labels(B, 1000, 1000)).pin_memory()
    hloss = torch.empty((), dtype=torch.float32).pin_memory()
    dstage = [torch.empty_like(net.a[0]) for _ in range(2)]
    cs = torch.cuda.Stream()
    copied = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]

    def run(h2d, dcopy, labels, loss):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)

        def prefetch(i):
            k = i % 2
            cs.wait_stream(stream) if i < 2 else cs.wait_event(consumed[k])
            with torch.cuda.stream(cs):
                dstage[k].copy_(hX, non_blocking=True)
                copied[k].record(cs)
        if h2d:
            prefetch(0)
        for i in range(K):
            k = i % 2
            if h2d:
                if i + 1 < K:
                    prefetch(i + 1)
                stream.wait_event(copied[k])
            if dcopy:
                net.a[0].copy_(dstage[k], non_blocking=True)
                consumed[k].record(stream)
            if labels:
                net.labels.copy_(hL, non_blocking=True)
            g.replay()
            if loss:
                hloss.copy_(net.loss, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    # host pack: the first layer's packed operand is built straight from the pinned int8 host batch
    # by the pack kernel (zero-copy reads over PCIe) on the copy stream, into the workspace of the
    # other of two captured graphs (external_pack: the graphs do not pack)
    import paper_1408_5093_b200 as cb
    L0 = net.layers[0]
    ws0s = [net.ws0, cb.conv_bottom_workspace(net.shapes[0], tuple(net.W[0].shape), L0.stride, L0.pad, L0.group,
                                              "bf16", dev)]
    net.external_pack = True
    hgraphs = []
    for k in range(2):
        net.ws0 = ws0s[k]
        hgraphs.append(net.capture())
    net.ws0 = ws0s[0]
    net.external_pack = False

    def run_hostpack():
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)

        def pack(i):
            k = i % 2
            cs.wait_stream(stream) if i < 2 else cs.wait_event(consumed[k])
            with torch.cuda.stream(cs):
                cb.conv_pack_bottom(hX, net._wop(0), L0.stride, L0.pad, L0.group, "bf16", ws=ws0s[k])
                copied[k].record(cs)
        pack(0)
        for i in range(K):
            k = i % 2
            if i + 1 < K:
                pack(i + 1)
            stream.wait_event(copied[k])
            net.labels.copy_(hL, non_blocking=True)
            hgraphs[k].replay()
            consumed[k].record(stream)
            hloss.copy_(net.loss, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    import statistics
    cfgs = [("full", (1, 1, 1, 1)), ("no_h2d", (0, 1, 1, 1)), ("replay_only", (0, 0, 0, 0)), ("hostpack", None)]
    res = {n: [] for n, _ in cfgs}
    for _ in range(6):
        for name, cfg in cfgs:
            res[name].append(run(*cfg) if cfg is not None else run_hostpack())
    for name, _ in cfgs:
        print(f"{name:16s} median {statistics.median(res[name]):.4f} ms/step  {['%.3f' % x for x in res[name]]}",
              flush=True)


if __name__ == "__main__":
    main()
