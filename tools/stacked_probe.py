import sys, os, torch
sys.path.insert(0, 'tools'); sys.path.insert(0, '.')
import paper_1408_5093_b200 as cb
from paper_1408_5093_b200 import _abi
from gemm_probe import timeit
dev = torch.device("cuda"); B = 256; cl = torch.channels_last
def T(*s): return torch.randn(*s, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
cases = {"conv3": (256, 384, 1), "conv4": (384, 384, 2), "conv5": (384, 256, 2)}
for mode, ast in ((0, 2), (2, 2)):
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_STACKED, mode)
    out = []
    for name, (C, O, g) in cases.items():
        x = T(B, C, 13, 13); w = (torch.randn(O, C // g, 3, 3, device=dev) * 0.01).to(torch.bfloat16)
        bb = torch.zeros(O, device=dev); y = T(B, O, 13, 13); dy = T(B, O, 13, 13); dx = T(B, C, 13, 13)
        tf = timeit(lambda: cb.conv_forward(x, w, bb, 1, 1, g, "bf16", relu=True, out=y))
        td = timeit(lambda: cb.conv_backward_data(dy, w, x.shape, 1, 1, g, "bf16", out=dx))
        out.append(f"{name} fwd {tf*1e3:6.1f} dgrad {td*1e3:6.1f}")
    print("stacked", mode, "a_stages", ast, " | ".join(out), flush=True)
# conv2 forced
x2 = T(B, 96, 27, 27); w2 = (torch.randn(256, 48, 5, 5, device=dev) * 0.01).to(torch.bfloat16); b2 = torch.zeros(256, device=dev)
y2 = T(B, 256, 27, 27); dy2 = T(B, 256, 27, 27); dx2 = T(B, 96, 27, 27)
for mode in (1, 2):
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_STACKED, mode)
    tf = timeit(lambda: cb.conv_forward(x2, w2, b2, 1, 2, 2, "bf16", relu=True, out=y2))
    td = timeit(lambda: cb.conv_backward_data(dy2, w2, x2.shape, 1, 2, 2, "bf16", out=dx2))
    print("conv2 stacked", mode, f"fwd {tf*1e3:6.1f} dgrad {td*1e3:6.1f}", flush=True)
