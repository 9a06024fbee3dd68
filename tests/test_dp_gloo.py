"""Data-parallel host logic on CPU (world size 2, gloo): bucketed asynchronous gradient allreduce of
the flat gradient buffer (paper_1408_5093_b200.dp) makes W x B/W-image steps equal one B-image step
(S:293 batch decomposability + reading R17), and leaves the replicas' parameters bit-identical."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layout(params, order):
    segs, off = [], 0
    for name in order:
        W, b = params[name]
        n = W.size + b.size
        segs.append((name, off, n))
        off = (off + n + 63) // 64 * 64
    return segs, off


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from oracle import net as onet
        import synth
        from paper_1408_5093_b200.dp import GradAllReduce
        oracle.build()
        B = 4
        X = synth.mnist_pixels((B, 1, 28, 28), 7)
        lab = synth.labels(B, 10, 7)

        def rng_w(name, shape, kind):
            return synth.xavier(shape, 3, synth.S_W, len(name)).astype(np.float64) if kind == "w" else \
                synth.uniform(shape, 3, synth.S_B, len(name)).astype(np.float64) * 0.1

        params = onet.init_params(onet.LENET, X.shape, rng_w)
        order = [name for kind, name, _ in onet.LENET if kind in ("conv", "ip")]
        segs, total = _layout(params, order)
        # this rank's shard of the batch
        sl = slice(rank * B // world, (rank + 1) * B // world)
        _, grads, _ = onet.forward_backward(onet.LENET, X[sl], params, lab[sl])
        flat = torch.zeros(total, dtype=torch.float64)
        ar = GradAllReduce(flat, segs, world, bucket_bytes=8 << 10)
        assert len(ar.buckets) >= 2
        for name in reversed(order):   # backward order
            dW, db = grads[name]
            off = dict((k, o) for k, o, _ in segs)[name]
            flat[off:off + dW.size] = torch.from_numpy(dW.ravel())
            flat[off + dW.size:off + dW.size + db.size] = torch.from_numpy(db.ravel())
            ar.on_grad(name)
        ar.finish()
        flat /= world
        # single-process reference on the full batch
        _, gfull, _ = onet.forward_backward(onet.LENET, X, params, lab)
        err = 0.0
        for name in order:
            dW, db = gfull[name]
            off = dict((k, o) for k, o, _ in segs)[name]
            got = flat[off:off + dW.size + db.size].numpy()
            want = np.concatenate([dW.ravel(), db.ravel()])
            err = max(err, float(np.max(np.abs(got - want))))
        # replicas identical after the exchange
        allf = [torch.zeros_like(flat) for _ in range(world)]
        dist.all_gather(allf, flat)
        same = all(torch.equal(allf[0], t) for t in allf)
        q.put((rank, err, same))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), False))


def test_dp_bucketed_allreduce_matches_full_batch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, same in res:
        assert not isinstance(err, str), err
        assert err < 1e-12, (rank, err)
        assert same


def test_bucket_tiling():
    from paper_1408_5093_b200.dp import GradAllReduce
    flat = torch.zeros(1000)
    segs = [("a", 0, 100), ("b", 128, 300), ("c", 448, 500), ("d", 960, 40)]
    ar = GradAllReduce(flat, segs, 2, bucket_bytes=1200)
    # buckets tile [0, 1000) with no gap, highest offsets first (backward order)
    assert ar.buckets[0][1] == 1000 and ar.buckets[-1][0] == 0
    for (lo1, hi1, _), (lo2, hi2, _) in zip(ar.buckets, ar.buckets[1:]):
        assert lo1 == hi2
    keys = set().union(*[b[2] for b in ar.buckets])
    assert keys == {"a", "b", "c", "d"}
