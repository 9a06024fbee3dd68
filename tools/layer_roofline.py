"""Per-pass roofline table of the CaffeNet training step at batch 256 (BF16, channels-last, the
library's default kernels): every convolution / inner-product pass and the bandwidth layers timed
ALONE with CUDA events over graph-captured repeats, warm (back to back) and cold (an L2 flush of
512 MB before every call, its own time subtracted), against the algorithmic work of SURVEY App. A
(FLOPs = 2*MACs; bytes = each tensor read or written once, U8 pool masks) and MEASURED_PEAKS.json
(burst BF16 tensor peak, HBM copy bandwidth).

    python tools/layer_roofline.py [--json out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = 256
CL = torch.channels_last
dev = torch.device("cuda")


def bf(shape, scale=1.0):
    return (torch.randn(*shape, device=dev) * scale).to(torch.bfloat16).contiguous(memory_format=CL)


def graph_time(fn, inner=10, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(inner):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) / inner)
    return sorted(ts)[reps // 2]   # ms


FLUSH = None


def flush():
    FLUSH.zero_()


def timed(fn):
    warm = graph_time(fn)
    cold = graph_time(lambda: (flush(), fn())) - graph_time(flush)
    return warm, cold


def main():
    global FLUSH
    FLUSH = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    tc_peak, hbm = peaks["bf16_tflops"], peaks["hbm_gbs"]
    rows = []

    def add(name, fn, gflop=0.0, mb=0.0):
        w, c = timed(fn)
        r = {"pass": name, "warm_us": round(w * 1e3, 2), "cold_us": round(c * 1e3, 2)}
        if gflop:
            r.update(gflop=round(gflop, 2), tflops=round(gflop / w, 1), frac_tensor=round(gflop / w / tc_peak, 3))
        if mb:
            r.update(mb=round(mb, 1), gbs=round(mb / w, 0), frac_hbm=round(mb / w / hbm, 3))
        rows.append(r)
        print(json.dumps(r), flush=True)

    conv = [("conv1", 3, 227, 96, 11, 4, 0, 1), ("conv2", 96, 27, 256, 5, 1, 2, 2), ("conv3", 256, 13, 384, 3, 1, 1, 1),
            ("conv4", 384, 13, 384, 3, 1, 1, 2), ("conv5", 384, 13, 256, 3, 1, 1, 2)]
    for name, C, H, O, k, s, p, g in conv:
        OH = (H + 2 * p - k) // s + 1
        gf = 2.0 * B * OH * OH * O * (C // g) * k * k / 1e9
        if C == 3:
            x = torch.randint(-128, 128, (B, C, H, H), device=dev).to(torch.bfloat16).contiguous(memory_format=CL)
        else:
            x = bf((B, C, H, H))
        w = (torch.randn(O, C // g, k, k, device=dev) * 0.01).to(torch.bfloat16)
        b = torch.zeros(O, device=dev)
        y = torch.empty(B, O, OH, OH, device=dev, dtype=torch.bfloat16).contiguous(memory_format=CL)
        dy = bf((B, O, OH, OH))
        dw = torch.zeros(O, C // g, k, k, device=dev)
        db = torch.zeros(O, device=dev)
        if C == 3:   # the net packs the image batch once per step (space-to-depth) for fwd + wgrad
            wsb = cb.conv_bottom_workspace(x.shape, w.shape, s, p, g, "bf16", dev)
            cb.conv_pack_bottom(x, w, s, p, g, "bf16", ws=wsb)
            add(f"{name} fwd", lambda: cb.conv_forward(x, w, b, s, p, g, "bf16", relu=True, out=y, ws=wsb,
                                                       prepacked=True), gf)
            add(f"{name} wgrad", lambda: cb.conv_backward_weight(x, dy, w.shape, s, p, g, "bf16", dw=dw, db=db,
                                                                 ws=wsb, prepacked=True), gf)
            continue
        wsf = cb.conv_workspace(x.shape, w.shape, s, p, g, "bf16", 0, dev)
        wsd = cb.conv_workspace(x.shape, w.shape, s, p, g, "bf16", 1, dev)
        wsw = cb.conv_workspace(x.shape, w.shape, s, p, g, "bf16", 2, dev)
        dx = torch.empty_like(x)
        add(f"{name} fwd", lambda: cb.conv_forward(x, w, b, s, p, g, "bf16", relu=True, out=y, ws=wsf), gf)
        add(f"{name} dgrad", lambda: cb.conv_backward_data(dy, w, x.shape, s, p, g, "bf16", out=dx, ws=wsd), gf)
        add(f"{name} wgrad", lambda: cb.conv_backward_weight(x, dy, w.shape, s, p, g, "bf16", dw=dw, db=db, ws=wsw), gf)

    for name, K, O in [("fc6", 9216, 4096), ("fc7", 4096, 4096), ("fc8", 4096, 1000)]:
        gf = 2.0 * B * K * O / 1e9
        x = (torch.randn(B, K, device=dev)).to(torch.bfloat16)
        w = (torch.randn(O, K, device=dev) * 0.005).to(torch.bfloat16)
        b = torch.zeros(O, device=dev)
        y = torch.empty(B, O, device=dev, dtype=torch.bfloat16)
        dy = torch.randn(B, O, device=dev).to(torch.bfloat16)
        dx = torch.empty(B, K, device=dev, dtype=torch.bfloat16)
        dw = torch.zeros(O, K, device=dev)
        db = torch.zeros(O, device=dev)
        wmb = O * K * 2 / 1e6
        add(f"{name} fwd", lambda: cb.ip_forward(x, w, b, "bf16", relu=name != "fc8", out=y), gf, wmb)
        add(f"{name} dgrad", lambda: cb.ip_backward_data(dy, w, x.shape, "bf16", out=dx), gf, wmb)
        add(f"{name} wgrad", lambda: cb.ip_backward_weight(x, dy, w.shape, "bf16", dw=dw, db=db), gf, O * K * 4 / 1e6)

    # bandwidth layers (BF16 channels-last, U8 window-local masks)
    p1in = torch.relu(bf((B, 96, 55, 55)))
    p1 = torch.empty(B, 96, 27, 27, device=dev, dtype=torch.bfloat16).contiguous(memory_format=CL)
    m1 = torch.empty(B, 96, 27, 27, device=dev, dtype=torch.uint8).contiguous(memory_format=CL)
    n1 = torch.empty_like(p1)
    add("pool1 fwd", lambda: cb.pool_forward(p1in, "max", 3, 2, out=p1, mask=m1), 0, (148.7 + 35.8 + 17.9))
    add("norm1 fwd", lambda: cb.lrn_forward(p1, out=n1), 0, 2 * 35.8)
    dn1 = bf((B, 96, 27, 27))
    dp1 = torch.empty_like(p1)
    add("norm1 bwd", lambda: cb.lrn_backward(p1, n1, dn1, out=dp1), 0, 3 * 35.8)
    dc1 = torch.empty_like(p1in)
    add("pool1+relu1 bwd", lambda: cb.pool_relu_backward(p1, dp1, m1, p1in.shape, 3, 2, out=dc1), 0,
        35.8 + 17.9 + 35.8 + 148.7)
    p2in = torch.relu(bf((B, 256, 27, 27)))
    p2 = torch.empty(B, 256, 13, 13, device=dev, dtype=torch.bfloat16).contiguous(memory_format=CL)
    m2 = torch.empty(B, 256, 13, 13, device=dev, dtype=torch.uint8).contiguous(memory_format=CL)
    n2 = torch.empty_like(p2)
    add("pool2+norm2 fwd (fused)", lambda: cb.pool_lrn_forward(p2in, 3, 2, pool_out=p2, mask=m2, out=n2), 0,
        95.6 + 22.2 + 11.1 + 22.2)
    dn2 = bf((B, 256, 13, 13))
    dp2 = torch.empty_like(p2)
    add("norm2 bwd", lambda: cb.lrn_backward(p2, n2, dn2, out=dp2), 0, 3 * 22.2)
    dc2 = torch.empty_like(p2in)
    add("pool2+relu2 bwd", lambda: cb.pool_relu_backward(p2, dp2, m2, p2in.shape, 3, 2, out=dc2), 0,
        22.2 + 11.1 + 22.2 + 95.6)
    n = 60965224
    wp = torch.randn(n, device=dev)
    gp = torch.randn(n, device=dev)
    vp = torch.zeros(n, device=dev)
    wq = torch.empty(n, device=dev, dtype=torch.bfloat16)
    add("sgd update (61 M params)", lambda: cb.sgd_update(wp, gp, vp, 0.01, 0.9, 5e-4, w_bf16=wq), 0, n * 22 / 1e6)
    conv_rows = [r for r in rows if r["pass"].startswith("conv")]
    gsum = sum(r["gflop"] for r in conv_rows)
    wsum = sum(r["warm_us"] for r in conv_rows)
    csum = sum(r["cold_us"] for r in conv_rows)
    summary = {"conv_gflop": round(gsum, 2), "conv_warm_us": round(wsum, 1), "conv_cold_us": round(csum, 1),
               "conv_tflops_warm": round(gsum / wsum * 1e3, 1), "conv_frac_warm": round(gsum / wsum * 1e3 / tc_peak, 3),
               "conv_frac_cold": round(gsum / csum * 1e3 / tc_peak, 3), "peaks": {"bf16_tflops": tc_peak, "hbm_gbs": hbm},
               "note": "conv wgrad/dgrad times include their weight repacks and split reductions (the whole ABI call); "
                       "conv1 fwd/wgrad read the space-to-depth image batch packed once per step"}
    print(json.dumps(summary), flush=True)
    if "--json" in sys.argv:
        json.dump({"rows": rows, "summary": summary}, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
