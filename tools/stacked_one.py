"""One stacked-halo conv3 forward (CaffeNet shape, CAFFE_TUNE_HALO_STACKED=2) for ncu."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1408_5093_b200 as cb
from paper_1408_5093_b200 import _abi
dev = torch.device("cuda"); B = 256; cl = torch.channels_last
x = torch.randn(B, 256, 13, 13, device=dev).to(torch.bfloat16).contiguous(memory_format=cl)
w = (torch.randn(384, 256, 3, 3, device=dev) * 0.01).to(torch.bfloat16)
bb = torch.zeros(384, device=dev)
y = torch.empty((B, 384, 13, 13), device=dev, dtype=torch.bfloat16).contiguous(memory_format=cl)
_abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_HALO_STACKED, int(sys.argv[1]) if len(sys.argv) > 1 else 2)
for _ in range(3):
    cb.conv_forward(x, w, bb, 1, 1, 1, "bf16", relu=True, out=y)
torch.cuda.synchronize()
