"""Micro-benchmark of the tcgen05 GEMM paths (run on the B200 box).

Times single ABI calls with CUDA events (median of 20 after warm-up) and prints TFLOP/s:
plain 2-D-tiled GEMMs through caffe_ip_forward and the CaffeNet conv passes with channels-last
BF16 operands (TMA im2col).
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1408_5093_b200 as cb  # noqa: E402


def timeit(fn, reps=5, inner=20):
    """Median over `reps` of the mean time of `inner` back-to-back calls captured in a CUDA graph
    (so host launch overhead does not leak into the device time)."""
    for _ in range(3):
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
    ts.sort()
    return ts[len(ts) // 2]


def main():
    torch.manual_seed(0)
    dev = torch.device("cuda")
    out = {}
    if "--spin" in sys.argv:
        from paper_1408_5093_b200 import _abi
        _abi.call("caffe_set_tuning", 2, int(sys.argv[sys.argv.index("--spin") + 1]))
    if "--halo" in sys.argv:
        from paper_1408_5093_b200 import _abi
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO, int(sys.argv[sys.argv.index("--halo") + 1]))
    if "--macc" in sys.argv:
        from paper_1408_5093_b200 import _abi
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_WGRAD_MACC, int(sys.argv[sys.argv.index("--macc") + 1]))
    if "--cta" in sys.argv:
        from paper_1408_5093_b200 import _abi
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_CTA_PAIR, int(sys.argv[sys.argv.index("--cta") + 1]))
    if "--only-conv3" in sys.argv:  # for ncu: a few launches of conv3 forward
        cl = torch.channels_last
        x = torch.randn(256, 256, 13, 13, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
        w = torch.randn(384, 256, 3, 3, device=dev) * 0.05
        y = cb.conv_forward(x, w, None, 1, 1, 1, relu=True)
        for _ in range(3):
            cb.conv_forward(x, w, None, 1, 1, 1, relu=True, out=y)
        torch.cuda.synchronize()
        return
    if "--rows" in sys.argv:
        from paper_1408_5093_b200 import _abi
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_ROWS_EPILOGUE, int(sys.argv[sys.argv.index("--rows") + 1]))
    if "--only-conv1" in sys.argv:   # for ncu: conv1 forward (halo, s2d) with rows epilogue off then on
        from paper_1408_5093_b200 import _abi
        cl = torch.channels_last
        x = (torch.rand(256, 3, 227, 227, device=dev) * 255 - 128).round().to(torch.bfloat16).contiguous(memory_format=cl)
        w = torch.randn(96, 3, 11, 11, device=dev) * 0.01
        wb = w.to(torch.bfloat16)
        b = torch.zeros(96, device=dev)
        y = cb.conv_forward(x, wb, b, 4, 0, 1, relu=True)
        for mode in (0, 1):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_ROWS_EPILOGUE, mode)
            cb.conv_forward(x, wb, b, 4, 0, 1, relu=True, out=y)
        torch.cuda.synchronize()
        return
    if "--only-conv2" in sys.argv:   # for ncu: conv2 forward + data gradient
        cl = torch.channels_last
        x = torch.randn(256, 96, 27, 27, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
        w = torch.randn(256, 48, 5, 5, device=dev) * 0.05
        y = cb.conv_forward(x, w, None, 1, 2, 2, relu=True)
        dy = torch.randn_like(y)
        dx = torch.empty_like(x)
        for _ in range(2):
            cb.conv_forward(x, w, None, 1, 2, 2, relu=True, out=y)
            cb.conv_backward_data(dy, w, x.shape, 1, 2, 2, out=dx)
        torch.cuda.synchronize()
        return
    if "--only-fc6w" in sys.argv:   # for ncu: fc6 weight gradient / forward / data gradient
        x = torch.randn(256, 9216, device=dev).to(torch.bfloat16)
        w = torch.randn(4096, 9216, device=dev).to(torch.bfloat16) * 0.01
        dy = torch.randn(256, 4096, device=dev).to(torch.bfloat16)
        dw = torch.empty(4096, 9216, device=dev)
        db = torch.empty(4096, device=dev)
        y = torch.empty(256, 4096, device=dev, dtype=torch.bfloat16)
        dx = torch.empty(256, 9216, device=dev, dtype=torch.bfloat16)
        for _ in range(2):
            cb.ip_backward_weight(x, dy, w.shape, dw=dw, db=db)
            cb.ip_forward(x, w, None, relu=True, out=y)
            cb.ip_backward_data(dy, w, x.shape, out=dx)
        torch.cuda.synchronize()
        return
    if "--only-gemm" in sys.argv:   # for ncu: a few launches of one plain GEMM
        M, N, K = 65536, 256, 1152
        x = torch.randn(M, K, device=dev).to(torch.bfloat16)
        w = torch.randn(N, K, device=dev).to(torch.bfloat16)
        y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        for _ in range(4):
            cb.ip_forward(x, w, None, out=y)
        torch.cuda.synchronize()
        return
    for (M, N, K) in [(65536, 128, 1600), (65536, 256, 1152), (65536, 192, 1728), (256, 4096, 9216)]:
        x = torch.randn(M, K, device=dev).to(torch.bfloat16)
        w = torch.randn(N, K, device=dev).to(torch.bfloat16)
        y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        ms = timeit(lambda: cb.ip_forward(x, w, None, out=y))
        out[f"gemm M{M} N{N} K{K}"] = round(2 * M * N * K / ms / 1e9, 1)
    cl = torch.channels_last
    B = 256
    # CaffeNet fc layers (bf16 rows; NHWC pool5 bottom for fc6)
    for name, (K, O) in {"fc6": (9216, 4096), "fc7": (4096, 4096), "fc8": (4096, 1000)}.items():
        x = torch.randn(B, K, device=dev).to(torch.bfloat16)
        w = torch.randn(O, K, device=dev).to(torch.bfloat16) * 0.01
        bias = torch.zeros(O, device=dev)
        y = torch.empty(B, O, device=dev, dtype=torch.bfloat16)
        dy = torch.randn(B, O, device=dev).to(torch.bfloat16)
        dx = torch.empty(B, K, device=dev, dtype=torch.bfloat16)
        dw = torch.empty(O, K, device=dev)
        db = torch.empty(O, device=dev)
        flops = 2 * B * K * O
        ms = timeit(lambda: cb.ip_forward(x, w, bias, relu=True, out=y))
        ms_d = timeit(lambda: cb.ip_backward_data(dy, w, x.shape, out=dx))
        ms_w = timeit(lambda: cb.ip_backward_weight(x, dy, w.shape, dw=dw, db=db))
        out[name] = {"fwd_us": round(ms * 1e3, 1), "dgrad_us": round(ms_d * 1e3, 1), "wgrad_us": round(ms_w * 1e3, 1),
                     "fwd_tflops": round(flops / ms / 1e9, 1), "wgrad_tflops": round(flops / ms_w / 1e9, 1)}
    for name, (C, H, O, k, st, p, g) in {"conv1": (3, 227, 96, 11, 4, 0, 1), "conv2": (96, 27, 256, 5, 1, 2, 2),
                                         "conv3": (256, 13, 384, 3, 1, 1, 1), "conv4": (384, 13, 384, 3, 1, 1, 2),
                                         "conv5": (384, 13, 256, 3, 1, 1, 2)}.items():
        if "--only-fc" in sys.argv:
            break
        x = torch.randn(B, C, H, H, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
        w = torch.randn(O, C // g, k, k, device=dev) * 0.05
        bias = torch.zeros(O, device=dev)
        y = cb.conv_forward(x, w, bias, st, p, g, relu=True)
        OH = y.shape[2]
        flops = 2 * B * O * OH * OH * (C // g) * k * k
        ms = timeit(lambda: cb.conv_forward(x, w, bias, st, p, g, relu=True, out=y))
        dy = torch.randn_like(y)
        dxo = torch.empty_like(x)
        ms_d = timeit(lambda: cb.conv_backward_data(dy, w, x.shape, st, p, g, out=dxo)) if name != "conv1" else float("nan")
        dw = torch.zeros_like(w)
        db = torch.zeros(O, device=dev)
        ms_w = timeit(lambda: cb.conv_backward_weight(x, dy, w.shape, st, p, g, dw=dw, db=db))
        out[name] = {"fwd_tflops": round(flops / ms / 1e9, 1), "dgrad_tflops": round(flops / ms_d / 1e9, 1),
                     "wgrad_tflops": round(flops / ms_w / 1e9, 1), "fwd_us": round(ms * 1e3, 1),
                     "dgrad_us": round(ms_d * 1e3, 1), "wgrad_us": round(ms_w * 1e3, 1)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
