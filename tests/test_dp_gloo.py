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


def _sgd_worker(rank, world, port, mode, q):
    """One SGD iteration of LeNet with the exchange applying the update (dp.BucketedSGD): per
    bucket all-reduce + update, or reduce-scatter + update of this rank's slice + all-gather; the
    update itself is the oracle's S:523 step on the flat CPU buffers (the library SGD runs on the GPU
    path, tests/test_gpu_dp.py)."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from oracle import net as onet
        import synth
        from paper_1408_5093_b200.dp import BucketedSGD
        oracle.build()
        B = 4
        X = synth.mnist_pixels((B, 1, 28, 28), 8)
        lab = synth.labels(B, 10, 8)

        def rng_w(name, shape, kind):
            return synth.xavier(shape, 4, synth.S_W, len(name)).astype(np.float64) if kind == "w" else \
                synth.uniform(shape, 4, synth.S_B, len(name)).astype(np.float64) * 0.1

        params = onet.init_params(onet.LENET, X.shape, rng_w)
        order = [name for kind, name, _ in onet.LENET if kind in ("conv", "ip")]
        segs, total = _layout(params, order)
        offs = {k: o for k, o, _ in segs}

        P = torch.zeros(total, dtype=torch.float64)
        for name in order:
            W, b = params[name]
            P[offs[name]:offs[name] + W.size] = torch.from_numpy(W.ravel())
            P[offs[name] + W.size:offs[name] + W.size + b.size] = torch.from_numpy(b.ravel())
        V = torch.zeros_like(P)
        G = torch.zeros_like(P)
        P0 = P.clone()
        lr, mom, decay = 0.05, 0.9, 1e-3

        def update(lo, hi, gs):
            w, v = oracle.sgd_update(P[lo:hi].numpy(), G[lo:hi].numpy(), V[lo:hi].numpy(), lr, mom, decay, gs)
            P[lo:hi] = torch.from_numpy(w)
            V[lo:hi] = torch.from_numpy(v)

        sync = BucketedSGD(G, P, V, None, segs, world, rank, update, mode=mode, bucket_bytes=8 << 10)
        assert len(sync.buckets) >= 2
        sl = slice(rank * B // world, (rank + 1) * B // world)
        _, grads, _ = onet.forward_backward(onet.LENET, X[sl], params, lab[sl])
        for name in reversed(order):   # backward order: gradient enqueued, then the layer is done
            dW, db = grads[name]
            G[offs[name]:offs[name] + dW.size] = torch.from_numpy(dW.ravel())
            G[offs[name] + dW.size:offs[name] + dW.size + db.size] = torch.from_numpy(db.ravel())
            sync.on_grad(name)
            sync.on_done(name)
        sync.finish()
        # single-process reference: the full-batch gradient, one oracle SGD step of every parameter
        _, gfull, _ = onet.forward_backward(onet.LENET, X, params, lab)
        err = 0.0
        for name in order:
            dW, db = gfull[name]
            o = offs[name]
            g = np.concatenate([dW.ravel(), db.ravel()])
            w0 = P0[o:o + g.size].numpy()
            w1, _ = oracle.sgd_update(w0, g, np.zeros_like(g), lr, mom, decay)
            err = max(err, float(np.max(np.abs(P[o:o + g.size].numpy() - w1))))
        allp = [torch.zeros_like(P) for _ in range(world)]
        dist.all_gather(allp, P)
        same = all(torch.equal(allp[0], t) for t in allp)
        q.put((rank, err, same))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc(), False))


@pytest.mark.parametrize("mode", ["allreduce", "sharded"])
def test_dp_bucketed_sgd_matches_full_batch_step(mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sgd_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, err, same in res:
        assert not isinstance(err, str), err
        assert err < 1e-14, (rank, err)
        assert same


def test_sharded_slices_tile_each_bucket():
    from paper_1408_5093_b200.dp import BucketedSGD
    flat = torch.zeros(1024)
    segs = [("a", 0, 100), ("b", 128, 300), ("c", 448, 500), ("d", 960, 40)]
    for world in (1, 2, 4, 8):
        got = {}
        for r in range(world):
            s = BucketedSGD(flat, flat, flat, None, segs, world, r, None, mode="sharded", bucket_bytes=1200)
            for bi in range(len(s.buckets)):
                got.setdefault(bi, []).append(s._slice(bi))
        for bi, sl in got.items():
            lo, hi, _ = s.buckets[bi]
            assert sl[0][0] == lo and sl[-1][1] == hi
            for (a0, a1), (b0, b1) in zip(sl, sl[1:]):
                assert a1 == b0 and a1 - a0 == b1 - b0 and a0 % 4 == 0
    with pytest.raises(ValueError):
        BucketedSGD(flat, flat, flat, None, [("a", 0, 1000)], 3, 0, None, mode="sharded")
