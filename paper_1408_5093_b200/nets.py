"""Straight-line CaffeNet / LeNet training steps over the C ABI (host orchestration only).

The paper's nets (Fig. 1 LeNet; P:117-119 reference "AlexNet with variations",
i.e. CaffeNet) are linear chains, so the DAG bookkeeping of P:162-165 reduces to a fixed
call list.  Every layer call goes to libcaffe_b200.so; this module only allocates blobs,
wires them and orders the calls.

Layout: activations and their diffs in BF16 (or F32), parameters as one flat FP32 master
buffer (weights and biases), one flat FP32 gradient buffer (the data-parallel allreduce unit),
one flat FP32 momentum buffer and one flat BF16 copy of the weights consumed by the BF16
tensor-core operands.  The SGD update writes the BF16 copy as a side output.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

import paper_1408_5093_b200 as cb
from paper_1408_5093_b200 import _abi


@dataclass
class Layer:
    kind: str                 # conv | pool | lrn | ip | loss
    name: str
    num_output: int = 0
    kernel: int = 0
    stride: int = 1
    pad: int = 0
    group: int = 1
    relu: bool = False
    method: str = "max"
    w_std: float = 0.0        # gaussian std (0 -> xavier)
    b_init: float = 0.0


# CaffeNet (bvlc_reference_caffenet topology; SURVEY Sec. 8 shapes): conv1 -> relu1 -> pool1 -> norm1 ...
CAFFENET: List[Layer] = [
    Layer("conv", "conv1", 96, 11, 4, 0, 1, True, w_std=0.01, b_init=0.0),
    Layer("pool", "pool1", kernel=3, stride=2),
    Layer("lrn", "norm1"),
    Layer("conv", "conv2", 256, 5, 1, 2, 2, True, w_std=0.01, b_init=1.0),
    Layer("pool", "pool2", kernel=3, stride=2),
    Layer("lrn", "norm2"),
    Layer("conv", "conv3", 384, 3, 1, 1, 1, True, w_std=0.01, b_init=0.0),
    Layer("conv", "conv4", 384, 3, 1, 1, 2, True, w_std=0.01, b_init=1.0),
    Layer("conv", "conv5", 256, 3, 1, 1, 2, True, w_std=0.01, b_init=1.0),
    Layer("pool", "pool5", kernel=3, stride=2),
    Layer("ip", "fc6", 4096, relu=True, w_std=0.005, b_init=1.0),
    Layer("ip", "fc7", 4096, relu=True, w_std=0.005, b_init=1.0),
    Layer("ip", "fc8", 1000, w_std=0.01, b_init=0.0),
    Layer("loss", "loss"),
]
CAFFENET_INPUT = (3, 227, 227)

# LeNet (Fig. 1): conv1 20@5x5 -> pool 2x2/2 -> conv2 50@5x5 -> pool -> ip1 500 -> relu -> ip2 10
LENET: List[Layer] = [
    Layer("conv", "conv1", 20, 5, 1, 0, 1, False),
    Layer("pool", "pool1", kernel=2, stride=2),
    Layer("conv", "conv2", 50, 5, 1, 0, 1, False),
    Layer("pool", "pool2", kernel=2, stride=2),
    Layer("ip", "ip1", 500, relu=True),
    Layer("ip", "ip2", 10),
    Layer("loss", "loss"),
]
LENET_INPUT = (1, 28, 28)

LRN = dict(local_size=5, alpha=1e-4, beta=0.75, k=1.0)


def conv_flops(in_shape, L: Layer) -> Tuple[int, Tuple[int, int, int, int]]:
    """Algorithmic FLOPs of one conv pass (2 * MACs) and the output shape."""
    N, C, H, W = in_shape
    OH = (H + 2 * L.pad - L.kernel) // L.stride + 1
    OW = (W + 2 * L.pad - L.kernel) // L.stride + 1
    macs = N * L.num_output * OH * OW * (C // L.group) * L.kernel * L.kernel
    return 2 * macs, (N, L.num_output, OH, OW)


def torch_cuda_ok(net) -> bool:
    """Side streams need CUDA tensors (the CPU tests drive the oracle net, not this class)."""
    return net.params.is_cuda


class Net:
    def __init__(self, layers: List[Layer], batch: int, input_shape, device, act_dtype=None, math="bf16", seed=0,
                 input_i8=False):
        import torch
        import synth
        self.torch = torch
        self.layers = layers
        self.batch = batch
        self.device = device
        self.math = math
        self.act_dtype = act_dtype or (torch.bfloat16 if math == "bf16" else torch.float32)
        self.shapes = []            # input shape of each layer
        shape = (batch,) + tuple(input_shape)
        pspecs = []                 # (layer idx, w_shape, b_shape)
        self.hwc = {}               # inner products whose weight columns are stored in (h, w, c) order
        self.conv_flops_fwd = 0
        self.conv_flops_step = 0    # fwd + wgrad + dgrad (no dgrad for the first layer)
        for i, L in enumerate(layers):
            self.shapes.append(shape)
            if L.kind == "conv":
                f, out = conv_flops(shape, L)
                self.conv_flops_fwd += f
                self.conv_flops_step += 2 * f + (f if i > 0 else 0)
                pspecs.append((i, (L.num_output, shape[1] // L.group, L.kernel, L.kernel), (L.num_output,)))
                shape = out
            elif L.kind == "pool":
                shape = cb.pool_output_shape(shape, L.method, L.kernel, L.stride, L.pad)
            elif L.kind == "ip":
                K = int(np.prod(shape[1:]))
                pspecs.append((i, (L.num_output, K), (L.num_output,)))
                if self.fc_hwc and len(shape) == 4 and shape[2] * shape[3] > 1:
                    self.hwc[i] = (shape[1], shape[2], shape[3])
                shape = (batch, L.num_output)
            elif L.kind == "lrn":
                pass
        self.out_shape = shape
        # flat parameter storage: [w0, b0, w1, b1, ...]
        offs, total = [], 0
        for (_, ws, bs) in pspecs:
            nw, nb = int(np.prod(ws)), int(np.prod(bs))
            offs.append((total, nw, total + nw, nb))
            total += nw + nb
            total = (total + 63) // 64 * 64  # 256-byte alignment of every tensor
        self.nparams = total
        f32 = torch.float32
        self.params = torch.zeros(total, dtype=f32, device=device)
        self.grads = torch.zeros(total, dtype=f32, device=device)
        self.mom = torch.zeros(total, dtype=f32, device=device)
        self.params_bf16 = torch.zeros(total, dtype=torch.bfloat16, device=device)
        self.W, self.B, self.dW, self.dB, self.Wq, self.Mw = {}, {}, {}, {}, {}, {}
        host = np.zeros(total, np.float32)
        for k, ((i, ws, bs), (ow, nw, ob, nb)) in enumerate(zip(pspecs, offs)):
            L = layers[i]
            w = synth.gaussian(ws, L.w_std, seed, synth.S_W, k) if L.w_std > 0 else synth.xavier(ws, seed, synth.S_W, k)
            if i in self.hwc:   # the same weights, columns permuted from (c, h, w) to (h, w, c)
                C, H, Wd = self.hwc[i]
                w = w.reshape(ws[0], C, H, Wd).transpose(0, 2, 3, 1)
            host[ow:ow + nw] = w.ravel()
            host[ob:ob + nb] = L.b_init
            self.W[i] = self.params[ow:ow + nw].view(ws)
            self.B[i] = self.params[ob:ob + nb]
            self.dW[i] = self.grads[ow:ow + nw].view(ws)
            self.dB[i] = self.grads[ob:ob + nb]
            self.Wq[i] = self.params_bf16[ow:ow + nw].view(ws)
            self.Mw[i] = self.mom[ow:ow + nw].view(ws)
        # gradient segments (layer index, offset, numel incl. bias) for the data-parallel buckets
        self.segments = [(i, ow, ob + nb - ow) for (i, _, _), (ow, nw, ob, nb) in zip(pspecs, offs)]
        self.bias_seg = {i: (ob, nb) for (i, _, _), (ow, nw, ob, nb) in zip(pspecs, offs)}
        self.params.copy_(torch.from_numpy(host))
        self.params_bf16.copy_(self.params.to(torch.bfloat16))
        self.pspecs = pspecs
        # activations: a[i] = input of layer i; d[i] = diff w.r.t. a[i]
        self.a, self.d, self.mask = [], [], {}
        ad = self.act_dtype
        # every 4-D activation is channels-last (NHWC): the tensor-core conv reads and writes it
        # without a transpose and pool/LRN use 16-byte channel vectors; the inner product flattens
        # its NHWC input in the (c,h,w) order of S:130 inside the library.
        self.nhwc = [L.kind != "loss" and len(self.shapes[i]) == 4 for i, L in enumerate(layers)]
        # input_i8: the image batch is stored as int8 (integer pixels, e.g. mean-subtracted, exact in
        # BF16) and converted by the first layer's pack (CAFFE_I8): half the input bytes
        self.input_i8 = bool(input_i8 and math == "bf16" and layers[0].kind == "conv" and self.nhwc[0])
        for i, L in enumerate(layers):
            s = self.shapes[i]
            dt0 = torch.int8 if (i == 0 and self.input_i8) else ad
            self.a.append(cb.empty_like_layout(s, dt0, device, nhwc=self.nhwc[i]))
            self.d.append(cb.empty_like_layout(s, ad, device, nhwc=self.nhwc[i]) if i > 0 else None)
        self.scores = torch.empty(self.shapes[-1], dtype=torch.float32, device=device)
        # the loss gradient in the activation dtype: the softmax kernel writes the RNE BF16 value the
        # fc8 tensor-core passes would otherwise convert it to (no separate convert pass)
        self.dscores = torch.empty(self.shapes[-1], dtype=self.act_dtype, device=device)
        for i, L in enumerate(layers):
            if L.kind == "pool":
                # window-local uint8 argmax (a quarter of the int32 mask traffic; same results)
                self.mask[i] = cb.empty_like_layout(self.shapes[i + 1], torch.uint8, device, nhwc=self.nhwc[i + 1])
        # (an NCHW copy of fc6's channels-last input shared by its forward and weight gradient --
        # caffe_blob_to_nchw -- measured slower: 1.542 -> 1.572 ms/step; each pass stages its own)
        self.rows = {}
        self.labels = torch.zeros(batch, dtype=torch.int32, device=device)
        self.loss = torch.zeros((), dtype=torch.float32, device=device)
        # the first conv's operand (space-to-depth packed image batch) is built once per step into a
        # dedicated workspace and reused by its forward and weight-gradient passes
        self.ws0 = None
        if layers[0].kind == "conv" and math != "fp32":
            L0 = layers[0]
            self.ws0 = cb.conv_bottom_workspace(self.shapes[0], tuple(self.W[0].shape), L0.stride, L0.pad, L0.group,
                                                math, device)

        # conv weight operands packed once per weight change into dedicated per-layer workspaces
        # (caffe_conv_pack_weights + CAFFE_WEIGHTS_PREPACKED): the forward and data-gradient passes
        # then skip their per-call repack, and the repack runs right after each layer's update
        self.wsf, self.wsd = {}, {}
        if math != "fp32" and self.prepack_weights:
            for i, L in enumerate(layers):
                if L.kind != "conv":
                    continue
                ws_shape = tuple(self.W[i].shape)
                self.wsf[i] = (self.ws0 if (i == 0 and self.ws0 is not None) else
                               cb.conv_workspace(self.shapes[i], ws_shape, L.stride, L.pad, L.group, math, 0, device))
                if i > 0:
                    self.wsd[i] = cb.conv_workspace(self.shapes[i], ws_shape, L.stride, L.pad, L.group, math, 1, device)
                self.repack_weights(i)

    def repack_weights(self, i=None):
        """Rebuild the packed conv weight operands (all conv layers, or layer i) from the current
        weights; call after any change of the weights outside step()."""
        for j in ([i] if i is not None else list(self.wsf)):
            L = self.layers[j]
            self.cb_pack(j, L)

    def cb_pack(self, j, L):
        cb.conv_pack_weights(self._wop(j), self.shapes[j], L.stride, L.pad, L.group, self.math, 0, ws=self.wsf[j])
        if j in self.wsd:
            cb.conv_pack_weights(self._wop(j), self.shapes[j], L.stride, L.pad, L.group, self.math, 1, ws=self.wsd[j])

    # --------------------------------------------------------------- one training iteration
    # fc6 (an inner product over a channels-last 4-D activation) keeps its weight columns in the
    # (h, w, c) order of the activation's memory, so its input, its data gradient and its weight
    # gradient's input are the channels-last buffers read as rows: no (c, h, w) staging transpose in
    # the forward or the weight gradient, no channels-last scatter in the data gradient's split-K
    # reduce.  The same linear map (S:130's (c, h, w) flatten with the columns permuted once);
    # canonical(i, t) returns a weight-shaped tensor in the (c, h, w) column order.
    fc_hwc = False

    def _ip_rows(self, i, t):
        """Layer i's (N, C, H, W) channels-last input (or its diff) as (N, H*W*C) rows."""
        if i not in self.hwc:
            return t
        r = t.permute(0, 2, 3, 1).reshape(t.shape[0], -1)
        assert r.data_ptr() == t.data_ptr(), "fc_hwc needs a channels-last activation"
        return r

    def canonical(self, i, t):
        """A weight-shaped (O, K) tensor / array of layer i in the (c, h, w) column order of S:130."""
        if i not in self.hwc:
            return t
        C, H, Wd = self.hwc[i]
        if isinstance(t, np.ndarray):
            return np.ascontiguousarray(t.reshape(t.shape[0], H, Wd, C).transpose(0, 3, 1, 2)).reshape(t.shape[0], -1)
        return t.reshape(t.shape[0], H, Wd, C).permute(0, 3, 1, 2).reshape(t.shape[0], -1)

    def _wop(self, i):
        return self.Wq[i] if self.math == "bf16" else self.W[i]

    # CaffeNet's pool -> LRN blocks (pool1/norm1, pool2/norm2) as one fused kernel
    # (caffe_pool_lrn_forward; bit-identical to the separate calls).  Measured (batch 256, one B200,
    # tools/pool_lrn_probe.py): forward pool2+norm2 40.6 -> 29.5 us, pool1+norm1 50.4 -> 52.9 us.
    # The fused backward (caffe_lrn_pool_backward: the LRN's bottom diff never stored) is off by
    # default: the separate, strip-prefetching pool backward and the LRN backward are faster
    # (norm1 83 vs 134 us, norm2 57 vs 69 us) -- the fused kernel's per-lane LRN work per window
    # column needs ~120 registers, which caps it at 16 warps per SM, too few to hide its loads.
    fuse_pool_lrn = True
    fuse_pool_lrn_c16 = True   # pool1/norm1 too, through the 16-channel-lane kernel
    fuse_lrn_pool_backward = False

    def _pool_lrn(self, i):
        """True when pool layer i and the LRN layer i+1 run as one fused kernel."""
        if not self.fuse_pool_lrn or i + 1 >= len(self.layers) - 1:
            return False
        L, N = self.layers[i], self.layers[i + 1]
        if L.kind != "pool" or N.kind != "lrn" or L.method != "max" or (L.kernel, L.stride, L.pad) != (3, 2, 0):
            return False
        x = self.a[i]
        ok = (x.dtype == self.torch.bfloat16 and self.nhwc[i] and x.shape[1] % 8 == 0
              and 2 * (self.shapes[i + 1][2] - 1) + 3 <= x.shape[2] and x.shape[2] <= 2 * self.shapes[i + 1][2] + 1)
        # the 8-channel-lane fused forward keeps every lane busy only when C/8 divides 32 (pool2/norm2,
        # C = 256); C = 96 (pool1/norm1) runs the 16-channel-lane form (CAFFE_TUNE_POOL_LRN_C16)
        C = x.shape[1]
        return ok and (self.fuse_lrn_pool_backward or 32 % (C // 8) == 0 or (self.fuse_pool_lrn_c16 and C % 16 == 0))

    # conv weight operands packed at the start of each step on a side stream (1: the forward
    # operands, 2: forward and data-gradient operands) into dedicated workspaces; the passes then
    # skip their per-call repack (CAFFE_WEIGHTS_PREPACKED) and only wait for their layer's pack --
    # the five forward repacks (2.4-4 us each) leave the serial forward.  Measured (same box,
    # tools/sched_sweep.py, 6 alternations): 1 -> 1.490-1.515 ms/step (mean 1.500), 0 -> 1.492-1.533
    # (mean 1.513); 2 (the data-gradient packs too) was not better than 1.  Bit-identical.
    pack_side = 1

    def _pack_side_begin(self):
        torch = self.torch
        if getattr(self, "_psf", None) is None:
            self._psf, self._psd = {}, {}
            for i, L in enumerate(self.layers):
                if L.kind != "conv":
                    continue
                wsh = tuple(self.W[i].shape)
                self._psf[i] = (self.ws0 if (i == 0 and self.ws0 is not None) else
                                cb.conv_workspace(self.shapes[i], wsh, L.stride, L.pad, L.group, self.math, 0, self.device))
                if i > 0:
                    self._psd[i] = cb.conv_workspace(self.shapes[i], wsh, L.stride, L.pad, L.group, self.math, 1,
                                                     self.device)
            self._pstream = torch.cuda.Stream(priority=self.wgrad_priority)
        main = torch.cuda.current_stream()
        self._pstream.wait_stream(main)   # the previous step's updates are complete on main
        self._pev_f, self._pev_d = {}, {}
        with torch.cuda.stream(self._pstream):
            for i in self._psf:
                L = self.layers[i]
                cb.conv_pack_weights(self._wop(i), self.shapes[i], L.stride, L.pad, L.group, self.math, 0, ws=self._psf[i])
                self._pev_f[i] = torch.cuda.Event()
                self._pev_f[i].record(self._pstream)
            if self.pack_side >= 2:
                for i in self._psd:
                    L = self.layers[i]
                    cb.conv_pack_weights(self._wop(i), self.shapes[i], L.stride, L.pad, L.group, self.math, 1,
                                         ws=self._psd[i])
                    self._pev_d[i] = torch.cuda.Event()
                    self._pev_d[i].record(self._pstream)

    def forward(self):
        a, n = self.a, len(self.layers)
        skip = set()
        side_pack = bool(self.pack_side) and self.math != "fp32" and not self.wsf
        if side_pack:
            self._pack_side_begin()
        for i, L in enumerate(self.layers):
            if i in skip:
                continue
            x = a[i]
            nxt = a[i + 1] if i + 1 < n - 1 else None
            if L.kind == "conv":
                pre = i == 0 and self.ws0 is not None
                if pre and not self.external_pack:
                    cb.conv_pack_bottom(x, self._wop(i), L.stride, L.pad, L.group, self.math, ws=self.ws0)
                wpre = i in self.wsf
                wsf = self.wsf.get(i)
                if side_pack:
                    self.torch.cuda.current_stream().wait_event(self._pev_f[i])
                    wpre, wsf = True, self._psf[i]
                cb.conv_forward(x, self._wop(i), self.B[i], L.stride, L.pad, L.group, self.math, relu=L.relu, out=nxt,
                                ws=wsf if wpre else (self.ws0 if pre else None), prepacked=pre, wprepacked=wpre)
            elif L.kind == "pool" and self._pool_lrn(i):
                cb.pool_lrn_forward(x, L.kernel, L.stride, L.pad, **LRN, pool_out=nxt, mask=self.mask[i], out=a[i + 2])
                skip.add(i + 1)
            elif L.kind == "pool":
                cb.pool_forward(x, L.method, L.kernel, L.stride, L.pad, out=nxt, mask=self.mask[i])
            elif L.kind == "lrn":
                cb.lrn_forward(x, **LRN, out=nxt)
            elif L.kind == "ip":
                out = nxt if nxt is not None else self.scores
                if i in self.rows:
                    x = cb.to_nchw(x, out=self.rows[i])
                x = self._ip_rows(i, x)
                cb.ip_forward(x, self._wop(i), self.B[i], self.math, relu=L.relu, out=out.view(out.shape[0], -1))
            elif L.kind == "loss":
                cb.softmax_loss(self.scores, self.labels, loss=self.loss, diff=self.dscores)
        if side_pack:   # rejoin (the data-gradient packs finished long before)
            self.torch.cuda.current_stream().wait_stream(self._pstream)

    def _relu_fused(self, i):
        """True when layer i's ReLU backward is folded into the MAX-pool backward of layer i+1."""
        if i < 0 or i + 1 >= len(self.layers):
            return False
        L, P = self.layers[i], self.layers[i + 1]
        return L.kind in ("conv", "ip") and L.relu and P.kind == "pool" and P.method == "max"

    def _wgrad_workspace(self):
        """Dedicated workspace of the side-stream weight-gradient passes (largest conv layer i > 0
        or inner-product layer; the passes run one after another on that stream)."""
        if getattr(self, "_ws_wgrad", None) is None:
            n = 0
            for i, L in enumerate(self.layers):
                if L.kind == "ip":
                    v = cb.ctypes.c_size_t()
                    cb.call("caffe_ip_workspace_size", cb.MATH[self.math], _abi.Shape4(*cb._shape4(self.shapes[i])),
                            int(L.num_output), 2, cb.ctypes.byref(v))
                    n = max(n, v.value)
                if L.kind == "conv" and i > 0:
                    d = cb._conv_desc((L.kernel, L.kernel), L.stride, L.pad, L.group, self.math)
                    v = cb.ctypes.c_size_t()
                    cb.call("caffe_conv_workspace_size", cb.ctypes.byref(d), _abi.Shape4(*cb._shape4(self.shapes[i])),
                            _abi.Shape4(*cb._shape4(tuple(self.W[i].shape))), int(_abi.CAFFE_PASS_BACKWARD_WEIGHT),
                            cb.ctypes.byref(v))
                    n = max(n, v.value)
            self._ws_wgrad = self.torch.empty(n + 2048, dtype=self.torch.uint8, device=self.device)
        return self._ws_wgrad

    def _relu_into_dgrad(self, i):
        """True when the ReLU backward of layer i-1 is folded into layer i's data gradient
        (caffe_conv_backward_data_relu: conv3 -> relu3 -> conv4, conv4 -> relu4 -> conv5;
        caffe_ip_backward_data_relu: fc6 -> relu6 -> fc7, fc7 -> relu7 -> fc8)."""
        if i <= 0 or self.layers[i].kind not in ("conv", "ip"):
            return False
        if self.layers[i].kind == "ip" and not self.fuse_ip_relu:
            return False
        P = self.layers[i - 1]
        return P.kind in ("conv", "ip") and P.relu

    # launch each layer's data gradient (main stream, the critical path) before its weight gradient
    # (side stream) so the persistent data-gradient GEMM claims the SMs first.  Measured equal early in
    # round 2 (1534 vs 1537 us/step); with the taps-in-N data gradient and the side-stream weight packs
    # it wins a 6-run same-box A/B: 1.469-1.494 (mean 1.482) against 1.484-1.528 (mean 1.500) ms/step
    dgrad_first = True
    # the inner-product weight gradients on the weight-gradient stream (False: on the main stream)
    ip_wgrad_side = True
    # conv / inner-product layers (names, space-separated) whose weight gradient starts only after
    # their data gradient has completed (measured: conv2 / conv2-5 no better, fc6 or fc8 +70-90 us)
    wgrad_after_dgrad = ""
    # cap on the persistent grid of the weight-gradient GEMMs on their side stream (0 = every SM):
    # leaves SMs to the critical path (data gradients, pool/LRN backward) they run beside
    wgrad_max_ctas = 0

    def _side_grid(self):
        import contextlib
        if not self.wgrad_max_ctas:
            return contextlib.nullcontext()

        @contextlib.contextmanager
        def cap():
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, int(self.wgrad_max_ctas))
            try:
                yield
            finally:
                _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_MAX_CTAS, 0)
        return cap()

    def _sgd_fusable(self, i):
        """caffe_ip_backward_weight_sgd applies: BF16 math, fan-in a multiple of 32 (TMA boxes)."""
        return self.math == "bf16" and self.layers[i].kind == "ip" and self.W[i].shape[1] % 32 == 0

    def backward(self, hook=None, done_hook=None, wgrad_stream=None, fused_sgd=None):
        """Backward in reverse; `hook(i)` is called after layer i's parameter gradients are enqueued
        (data-parallel bucketing point), `done_hook(i)` once nothing later in the step reads layer
        i's parameters (after its data gradient; after its weight gradient for the first layer).
        wgrad_stream: the weight gradients of conv layers i > 0 run there, concurrently with the
        data gradient and the rest of the backward on the current stream (they share only reads);
        self.wgrad_done[i] is the event recorded after layer i's weight gradient."""
        a, d, n = self.a, self.d, len(self.layers)
        torch = self.torch
        self.wgrad_done = {}
        for i in range(n - 2, -1, -1):
            L = self.layers[i]
            dy = d[i + 1] if i + 1 < n - 1 else self.dscores
            y = a[i + 1] if i + 1 < n - 1 else self.scores
            if L.kind in ("conv", "ip") and L.relu and not self._relu_fused(i) and not self._relu_into_dgrad(i + 1):
                cb.relu_backward(y, dy, inplace=True)  # sign of the ReLU output == sign test on its input
            if L.kind == "conv":
                pre = i == 0 and self.ws0 is not None
                side = wgrad_stream is not None and i > 0
                if side:
                    ev = torch.cuda.Event()
                    ev.record(torch.cuda.current_stream())

                def wgrad():
                    if side:
                        wgrad_stream.wait_event(ev)
                        with torch.cuda.stream(wgrad_stream), self._side_grid():
                            cb.conv_backward_weight(a[i], dy, self.W[i].shape, L.stride, L.pad, L.group, self.math,
                                                    beta=0.0, dw=self.dW[i], db=self.dB[i], ws=self._wgrad_workspace())
                            self.wgrad_done[i] = torch.cuda.Event()
                            self.wgrad_done[i].record(wgrad_stream)
                    else:
                        cb.conv_backward_weight(a[i], dy, self.W[i].shape, L.stride, L.pad, L.group, self.math,
                                                beta=0.0, dw=self.dW[i], db=self.dB[i], ws=self.ws0 if pre else None,
                                                prepacked=pre)
                    if hook:
                        hook(i)

                def dgrad():
                    wpre = i in self.wsd
                    wsd = self.wsd.get(i)
                    if getattr(self, "_pev_d", None) and i in self._pev_d:
                        torch.cuda.current_stream().wait_event(self._pev_d[i])
                        wpre, wsd = True, self._psd[i]
                    if i > 0 and self._relu_into_dgrad(i):
                        cb.conv_backward_data_relu(dy, self._wop(i), a[i], L.stride, L.pad, L.group, self.math,
                                                   out=d[i], ws=wsd, wprepacked=wpre)
                    elif i > 0:
                        cb.conv_backward_data(dy, self._wop(i), a[i].shape, L.stride, L.pad, L.group, self.math,
                                              beta=0.0, out=d[i], ws=wsd, wprepacked=wpre)

                if side and L.name in self.wgrad_after_dgrad.split():
                    # this layer's weight gradient waits for its data gradient (the critical path's
                    # GEMM runs alone, then the weight gradient overlaps the bandwidth-bound passes)
                    dgrad()
                    ev = torch.cuda.Event()
                    ev.record(torch.cuda.current_stream())
                    wgrad()
                elif side and self.dgrad_first:   # the critical path's kernel claims the SMs first
                    dgrad()
                    wgrad()
                else:
                    wgrad()
                    dgrad()
                if done_hook:
                    done_hook(i)
            elif L.kind == "ip" and fused_sgd is not None and wgrad_stream is not None and self._sgd_fusable(i):
                # one GPU: the weight update is fused into the weight-gradient GEMM; it rewrites the
                # BF16 weights, so it follows this layer's data gradient
                dy2 = dy.view(dy.shape[0], -1)
                xi, di = self._ip_rows(i, a[i]), self._ip_rows(i, d[i])
                if i > 0 and self._relu_into_dgrad(i):
                    cb.ip_backward_data_relu(dy2, self._wop(i), xi, self.math, out=di)
                elif i > 0:
                    cb.ip_backward_data(dy2, self._wop(i), xi.shape, self.math, beta=0.0, out=di)
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream())
                wgrad_stream.wait_event(ev)
                with torch.cuda.stream(wgrad_stream):
                    cb.ip_backward_weight_sgd(self.rows.get(i, xi), dy2, self.W[i], self.Mw[i], self.Wq[i], fused_sgd["lr"],
                                              fused_sgd["momentum"], fused_sgd["decay"], 1.0, db=self.dB[i],
                                              ws=self._wgrad_workspace())
                    self.wgrad_done[i] = torch.cuda.Event()
                    self.wgrad_done[i].record(wgrad_stream)
                if done_hook:
                    done_hook(i)
            elif L.kind == "ip":
                dy2 = dy.view(dy.shape[0], -1)
                xi, di = self._ip_rows(i, a[i]), self._ip_rows(i, d[i])
                side = wgrad_stream is not None and self.ip_wgrad_side
                if side:
                    ev = torch.cuda.Event()
                    ev.record(torch.cuda.current_stream())

                def wgrad():
                    if side:
                        wgrad_stream.wait_event(ev)
                        with torch.cuda.stream(wgrad_stream), self._side_grid():
                            cb.ip_backward_weight(self.rows.get(i, xi), dy2, self.W[i].shape, self.math, beta=0.0,
                                                  dw=self.dW[i], db=self.dB[i], ws=self._wgrad_workspace())
                            self.wgrad_done[i] = torch.cuda.Event()
                            self.wgrad_done[i].record(wgrad_stream)
                    else:
                        cb.ip_backward_weight(self.rows.get(i, xi), dy2, self.W[i].shape, self.math, beta=0.0,
                                              dw=self.dW[i], db=self.dB[i])
                    if hook:
                        hook(i)

                def dgrad():
                    if i > 0 and self._relu_into_dgrad(i):
                        cb.ip_backward_data_relu(dy2, self._wop(i), xi, self.math, out=di)
                    elif i > 0:
                        cb.ip_backward_data(dy2, self._wop(i), xi.shape, self.math, beta=0.0, out=di)

                if side and L.name in self.wgrad_after_dgrad.split():
                    dgrad()
                    ev = torch.cuda.Event()
                    ev.record(torch.cuda.current_stream())
                    wgrad()
                elif side and self.dgrad_first:
                    dgrad()
                    wgrad()
                else:
                    wgrad()
                    dgrad()
                if done_hook:
                    done_hook(i)
            elif L.kind == "pool" and self._pool_lrn(i) and self.fuse_lrn_pool_backward:
                cb.lrn_pool_backward(a[i + 1], d[i + 2], self.mask[i], a[i].shape, L.kernel, L.stride, L.pad, **LRN,
                                     relu=self._relu_fused(i - 1), out=d[i])
            elif L.kind == "lrn" and i > 0 and self._pool_lrn(i - 1) and self.fuse_lrn_pool_backward:
                pass   # with the pool below, in one kernel
            elif L.kind == "pool":
                if self._relu_fused(i - 1):  # conv -> ReLU -> MAX pool: ReLU backward folded in
                    cb.pool_relu_backward(y, dy, self.mask[i], a[i].shape, L.kernel, L.stride, L.pad, out=d[i])
                else:
                    cb.pool_backward(dy, self.mask[i], a[i].shape, L.method, L.kernel, L.stride, L.pad, out=d[i])
            elif L.kind == "lrn":
                cb.lrn_backward(a[i], y, dy, **LRN, out=d[i])

    def update(self, lr=0.01, momentum=0.9, decay=5e-4, grad_scale=1.0, solver=None):
        self._sgd(0, self.nparams, lr, momentum, decay, grad_scale, solver)
        self.repack_weights()

    def _sgd(self, lo, hi, lr, momentum, decay, grad_scale, solver):
        """SGD update of the flat parameter range [lo, hi): fixed lr, or the solver's
        device-resident schedule and divergence guard (caffe_sgd_update_solver)."""
        wb = self.params_bf16[lo:hi] if self.math == "bf16" else None
        if solver is not None:
            solver.update(self.params[lo:hi], self.grads[lo:hi], self.mom[lo:hi], wb, grad_scale)
        else:
            cb.sgd_update(self.params[lo:hi], self.grads[lo:hi], self.mom[lo:hi], lr, momentum, decay, grad_scale,
                          w_bf16=wb)

    # the first layer's packed input (ws0) is written by the caller before the step
    # (conv_pack_bottom from the host batch, e.g. bench.py's end-to-end input pipeline)
    external_pack = False
    # measurement only: leave out the SGD updates of the overlapped step (tools/sched_sweep.py)
    skip_update = False
    side_sgd_blocks = 1
    side_sgd_threads = 256     # (2 x 128-thread blocks per SM measured the same: 1.503 vs 1.507 ms/step)
    # side-stream SGD updates of the layers whose gradients are final may be held back until the
    # backward pass reaches this layer index (None: each layer's update is launched as soon as its
    # gradients are final).  Measured (graph replay, one B200, ms/step): with the weight gradients
    # on the main stream, 1.758 immediate / 1.675 held to conv3 / 1.842 held to conv2; with them on
    # their side stream (wgrad_side), 1.624 immediate / 1.726 held to conv3; no update at all 1.537.
    sgd_flush_layer = None
    # conv weight gradients (layers > 0) on their own stream, concurrent with the data gradients
    wgrad_side = True
    # one GPU: the inner-product weight updates fused into their weight-gradient GEMMs
    # (caffe_ip_backward_weight_sgd; the gradient never reaches memory).  Off by default: measured
    # slower in the three-stream step (1.606 -> 1.691 ms/step) -- the fused fc6 pass is a persistent
    # GEMM that holds every SM for ~210 us beside the conv backward, where the separate update
    # kernel (one small block per SM) trickles alongside.
    fuse_ip_sgd = False
    fuse_ip_relu = True
    # conv weight operands packed after each update (caffe_conv_pack_weights) instead of inside every
    # forward / data-gradient call.  Off by default: measured slower in the step (1.534 -> 1.561
    # ms/step, A/B on one box) although each pass loses its repack launch.
    prepack_weights = False
    # CUDA stream priorities (lower = more urgent; 0 is the default, -3 the most urgent on B200):
    # the critical path first, then the weight gradients, the updates last.  Measured (graph replay,
    # ms/step): all equal 1.538; main -2 / weight gradients -1 / updates 0: 1.509; main -3 / -2 / 0:
    # 1.509; main -2 alone 1.592; weight gradients -1 alone 1.646.
    main_priority = -2
    wgrad_priority = -1
    sgd_priority = 0

    def step(self, allreduce=None, lr=0.01, momentum=0.9, decay=5e-4, overlap_update=True, solver=None):
        """One SGD iteration.  With `solver` (paper_1408_5093_b200.solver.Solver) the learning rate,
        momentum and decay come from it: the iteration's lr is computed on the device from its state
        after the loss (which also arms the divergence guard), and the iteration counter advances at
        the end of the step -- all inside a captured graph too."""
        if solver is not None:
            momentum, decay = solver.momentum, solver.decay
        self.forward()
        if solver is not None:
            if allreduce is not None and hasattr(allreduce, "reduce_loss"):
                allreduce.reduce_loss(self.loss)   # data parallel: one guard decision for all ranks
            solver.begin(self.loss)
        self._step_rest(allreduce, lr, momentum, decay, overlap_update, solver)
        if solver is not None:
            solver.end()

    def _step_rest(self, allreduce, lr, momentum, decay, overlap_update, solver):
        if allreduce is None and overlap_update:
            # Single GPU: each layer's SGD update runs on a side stream as soon as nothing later in the
            # step reads that layer's parameters, co-resident with the remaining backward GEMMs (the
            # update kernel asks for the max-shared carveout so an SM running it can still take a
            # 200 KB tensor-core CTA).  Measured 2.03 vs 2.10 ms/step (graph replay).
            torch = self.torch
            main = torch.cuda.current_stream()
            if getattr(self, "_side", None) is None:
                self._side = torch.cuda.Stream(priority=self.sgd_priority)
            seg = {i: (off, n) for (i, off, n) in self.segments}
            wb = self.params_bf16 if self.math == "bf16" else None
            pending = []
            flush_at = self.sgd_flush_layer
            if flush_at is None:
                flush_at = len(self.layers)

            wstream = None
            if self.wgrad_side:
                if getattr(self, "_wside", None) is None:
                    self._wside = torch.cuda.Stream(priority=self.wgrad_priority)
                wstream = self._wside

            launched = []

            fused = (dict(lr=lr, momentum=momentum, decay=decay)
                     if (self.fuse_ip_sgd and wstream is not None and solver is None) else None)

            def launch():
                launched.append(1)
                # pending (layer, lo, hi) ranges of the flat parameter buffer; adjacent ones are merged
                wev = [self.wgrad_done[i] for i, _, _ in pending if i in getattr(self, "wgrad_done", {})]
                layers_done = sorted({i for i, _, _ in pending})
                rng = sorted((lo, hi) for _, lo, hi in pending)
                pending.clear()
                runs = []
                for lo, hi in rng:
                    if runs and runs[-1][1] >= lo - 64:   # 256-byte alignment padding between tensors
                        runs[-1][1] = max(runs[-1][1], hi)
                    else:
                        runs.append([lo, hi])
                ev = torch.cuda.Event()
                ev.record(main)
                self._side.wait_event(ev)
                for e in wev:
                    self._side.wait_event(e)
                # one 256-thread block per SM: leaves registers / thread slots for the main stream
                _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_SGD_BLOCKS_PER_SM, self.side_sgd_blocks)
                _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_SGD_THREADS, self.side_sgd_threads)
                with torch.cuda.stream(self._side):
                    for lo, hi in runs:
                        self._sgd(lo, hi, lr, momentum, decay, 1.0, solver)
                    for i in layers_done:
                        if i in self.wsf:
                            self.repack_weights(i)
                _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_SGD_BLOCKS_PER_SM, 0)
                _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_SGD_THREADS, 0)

            def done(i):
                if getattr(self, "skip_update", False):
                    return
                if fused is not None and self._sgd_fusable(i):
                    ob, nb = self.bias_seg[i]          # weights already updated by the fused pass
                    pending.append((i, ob, ob + nb))
                else:
                    off, n = seg[i]
                    pending.append((i, off, off + n))
                if i <= flush_at:
                    launch()

            self.backward(done_hook=done, wgrad_stream=wstream, fused_sgd=fused)
            if pending:
                launch()
            if launched:
                main.wait_stream(self._side)
            if wstream is not None and self.wgrad_done:
                main.wait_stream(wstream)
            return
        if allreduce is not None and getattr(allreduce, "applies_update", False):
            # data parallel with the update inside the exchange (dp.BucketedSGD): per bucket, the
            # all-reduce (or reduce-scatter) is issued once its gradients are complete, and the update
            # (of the whole bucket, or of this rank's slice followed by an all-gather) once its layers'
            # data gradients no longer read the weights -- no update pass after the backward
            torch = self.torch
            main = torch.cuda.current_stream()
            if getattr(self, "_wside", None) is None:
                self._wside = torch.cuda.Stream(priority=self.wgrad_priority)
            if getattr(self, "_side", None) is None:
                self._side = torch.cuda.Stream(priority=self.sgd_priority)
            wstream = self._wside
            if allreduce.stream is None:
                allreduce.stream = self._side
            allreduce.update = lambda lo, hi, gs: self._sgd(lo, hi, lr, momentum, decay, gs, solver)

            def hook(i):
                ev = torch.cuda.Event()
                ev.record(main)
                wstream.wait_event(ev)
                with torch.cuda.stream(wstream):
                    allreduce.on_grad(i)

            self.backward(hook=hook, done_hook=allreduce.on_done, wgrad_stream=wstream)
            main.wait_stream(wstream)
            allreduce.finish()
            if self.wsf:
                self.repack_weights()
            return
        if allreduce is not None and self.wgrad_side and torch_cuda_ok(self):
            # data parallel: weight gradients on their stream as on one GPU; each bucket's all-reduce
            # is issued from that stream after it has also caught up with the main stream, so the
            # collective follows every gradient of the bucket (the layer-0 gradient runs on main)
            torch = self.torch
            main = torch.cuda.current_stream()
            if getattr(self, "_wside", None) is None:
                self._wside = torch.cuda.Stream(priority=self.wgrad_priority)
            wstream = self._wside

            def hook(i):
                ev = torch.cuda.Event()
                ev.record(main)
                wstream.wait_event(ev)
                with torch.cuda.stream(wstream):
                    allreduce.on_grad(i)

            self.backward(hook=hook, wgrad_stream=wstream)
            main.wait_stream(wstream)
            allreduce.finish()
            self.update(lr, momentum, decay, grad_scale=1.0 / allreduce.world, solver=solver)
            return
        self.backward(hook=allreduce.on_grad if allreduce else None)
        scale = 1.0
        if allreduce:
            allreduce.finish()
            scale = 1.0 / allreduce.world
        self.update(lr, momentum, decay, grad_scale=scale, solver=solver)

    def capture(self, prologue=None, **kw):
        """Record one whole training step (every library launch) into a CUDA graph; replaying it
        re-runs the identical kernel sequence on the same buffers without host launch overhead.
        Call after at least one eager step (so the cached workspace has reached its size)."""
        torch = self.torch
        # the critical path (forward, data gradients) is captured at the main priority; the weight-
        # gradient and update streams run at theirs (stream priorities are kept by graph kernel nodes)
        s = torch.cuda.Stream(priority=self.main_priority)
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                if prologue is not None:
                    prologue()
                self.step(**kw)
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g
        return g


class TrainLoop:
    """A CUDA-graph-captured training loop over a device-resident pool of batches (
    P:174 "Data are processed in mini-batches that pass through the network sequentially"): one
    graph per pool batch, each = copy that batch into the input blobs + the whole training step with
    the solver's device-side schedule and divergence guard.  Replaying the graphs in order runs the
    loop with no per-layer host launches; `run` records each iteration's loss on the device and
    checks the guard every `check_every` iterations (and at the end)."""

    def __init__(self, net: "Net", solver, images, labels):
        torch = net.torch
        self.net, self.solver = net, solver
        self.images = images          # device (P, B, C, H, W) in the input blob's dtype / layout
        self.labels = labels          # device (P, B) int32
        self.graphs = []
        x0, l0 = net.a[0], net.labels
        x0.copy_(images[0])
        l0.copy_(labels[0])
        # one eager step to size the cached workspaces and create the side streams, then undo it
        saved = (net.params.clone(), net.mom.clone(), net.params_bf16.clone(), solver.state.clone())
        net.step(solver=solver)
        torch.cuda.synchronize()
        net.params.copy_(saved[0])
        net.mom.copy_(saved[1])
        net.params_bf16.copy_(saved[2])
        solver.state.copy_(saved[3])
        for b in range(images.shape[0]):
            def pro(b=b):
                x0.copy_(images[b])
                l0.copy_(labels[b])
            self.graphs.append(net.capture(prologue=pro, solver=solver))
        torch.cuda.synchronize()

    def run(self, iters: int, start: int = 0, check_every: int = 100):
        torch = self.net.torch
        trace = torch.empty(iters, dtype=torch.float32, device=self.net.device)
        for i in range(iters):
            self.graphs[(start + i) % len(self.graphs)].replay()
            trace[i].copy_(self.net.loss)
            if (i + 1) % check_every == 0:
                self.solver.check()
        self.solver.check()
        return trace
