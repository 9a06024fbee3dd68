"""Time the fused pool+LRN kernels against the separate calls at CaffeNet's batch-256 geometries
(pool1/norm1 on 96x55x55, pool2/norm2 on 256x27x27), CUDA events per call, L2 not flushed.

    python tools/pool_lrn_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_5093_b200 as cb  # noqa: E402
from paper_1408_5093_b200 import _abi  # noqa: E402


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    cl = torch.channels_last
    for name, shape in (("pool1/norm1", (256, 96, 55, 55)), ("pool2/norm2", (256, 256, 27, 27))):
        x = torch.randn(shape, device="cuda").relu_().to(torch.bfloat16).contiguous(memory_format=cl)
        P, M = cb.pool_forward(x, "max", 3, 2, mask_dtype=torch.uint8)
        Y = cb.lrn_forward(P)
        G = torch.randn(tuple(P.shape), device="cuda").to(torch.bfloat16).contiguous(memory_format=cl)
        dP = torch.empty_like(P)
        dX = torch.empty_like(x)
        t_pf = timeit(lambda: cb.pool_forward(x, "max", 3, 2, out=P, mask=M))
        t_lf = timeit(lambda: cb.lrn_forward(P, out=Y))
        t_ff = timeit(lambda: cb.pool_lrn_forward(x, pool_out=P, mask=M, out=Y))
        t_lb = timeit(lambda: cb.lrn_backward(P, Y, G, out=dP))
        t_pb = timeit(lambda: cb.pool_relu_backward(P, dP, M, x.shape, 3, 2, out=dX))
        res = {}
        for rb in (0, 1, 2, 4):
            _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_FUSED_POOL_ROWS, rb)
            res[rb] = timeit(lambda: cb.lrn_pool_backward(P, G, M, x.shape, out=dX))
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_FUSED_POOL_ROWS, 0)
        print(f"{name}: fwd separate {t_pf:.1f} + {t_lf:.1f} = {t_pf + t_lf:.1f} us, fused {t_ff:.1f} us | "
              f"bwd separate {t_lb:.1f} + {t_pb:.1f} = {t_lb + t_pb:.1f} us, fused " +
              " ".join(f"rb{k}={v:.1f}" for k, v in res.items()))


if __name__ == "__main__":
    main()


def step_times():
    """Whole CaffeNet step (graph replay, batch 256) with the pool+LRN blocks fused or separate."""
    import synth
    from paper_1408_5093_b200 import nets
    dev = torch.device("cuda")
    out = {}
    for fuse, rb in ((False, 0), (True, -1), (True, 2)):
        _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_FUSED_POOL_ROWS, max(rb, 0))
        net = nets.Net(nets.CAFFENET, 256, nets.CAFFENET_INPUT, dev, math="bf16", seed=0, input_i8=True)
        net.fuse_pool_lrn = fuse
        net.fuse_lrn_pool_backward = rb >= 0    # rb -1: fused forward only
        net.a[0].copy_(torch.from_numpy(synth.int_pixels((256, 3, 227, 227), 1000)).to(net.a[0].dtype))
        net.labels.copy_(torch.from_numpy(synth.labels(256, 1000, 1000)))
        for _ in range(3):
            net.step()
        torch.cuda.synchronize()
        net.capture()
        out[(fuse, rb)] = timeit(lambda: net.graph.replay(), reps=20)
        del net
        torch.cuda.empty_cache()
    _abi.call("caffe_set_tuning", _abi.CAFFE_TUNE_FUSED_POOL_ROWS, 0)
    print("step us: " + " ".join(f"{'fused' if f else 'separate'}{'_rb%d' % r if f else ''}={v:.1f}"
                                 for (f, r), v in out.items()))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "step":
    step_times()
