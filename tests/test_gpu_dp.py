"""Data-parallel training step through the library (-m gpu).

* world size 2 on ONE GPU (two processes, gloo over CUDA tensors -- NCCL refuses two ranks on one
  device): Net.step with the bucketed all-reduce (update after the exchange), with the per-bucket
  all-reduce + update (dp.BucketedSGD "allreduce") and with reduce-scatter + sharded SGD +
  all-gather (dp.BucketedSGD "sharded") each match the single-process step on the concatenated
  2B-image batch (S:293 batch decomposability, reading R17), and leave both replicas' parameters
  bit-identical.  The two ranks get different images, so an exchange that ran before the gradients
  were final, or an update that missed a bucket, changes the result.
* world size 1 NCCL: every exchange mode equals the serial step bit for bit, eager and captured in
  a CUDA graph (the collectives inside the graph).
"""
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

B = 8
MODES = ["grad_allreduce", "allreduce", "sharded"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _make_net(batch, seed=5):
    import torch
    from paper_1408_5093_b200 import nets
    return nets.Net(nets.LENET, batch, nets.LENET_INPUT, torch.device("cuda", 0), math="bf16", seed=seed)


def _batch(n0, n):
    X = synth.mnist_pixels((16,) + (1, 28, 28), 21)[n0:n0 + n]
    lab = synth.labels(16, 10, 21)[n0:n0 + n]
    return X, lab


def _sync(mode, net, world, rank, group=None):
    from paper_1408_5093_b200.dp import BucketedSGD, GradAllReduce
    if mode == "grad_allreduce":
        return GradAllReduce(net.grads, net.segments, world, bucket_bytes=64 << 10, group=group)
    return BucketedSGD(net.grads, net.params, net.mom, net.params_bf16, net.segments, world, rank, mode=mode,
                       bucket_bytes=64 << 10, group=group)


def _worker(rank, world, port, mode, out):
    import torch
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        net = _make_net(B)
        X, lab = _batch(rank * B, B)
        net.a[0].copy_(torch.from_numpy(X).to(net.a[0].dtype))
        net.labels.copy_(torch.from_numpy(lab))
        sync = _sync(mode, net, world, rank)
        for _ in range(2):
            net.step(sync)
        torch.cuda.synchronize()
        np.save(out + f".{rank}.npy", net.params.cpu().numpy())
        np.save(out + f".{rank}.bf16.npy", net.params_bf16.float().cpu().numpy())
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        with open(out + f".{rank}.err", "w") as f:
            f.write(traceback.format_exc())


@pytest.mark.parametrize("mode", MODES)
def test_dp_world2_one_gpu_matches_full_batch(tmp_path, mode):
    import torch
    import torch.multiprocessing as mp
    world = 2
    out = str(tmp_path / "p")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    for r in range(world):
        if os.path.exists(out + f".{r}.err"):
            pytest.fail(open(out + f".{r}.err").read())
    got = [np.load(out + f".{r}.npy") for r in range(world)]
    gotb = [np.load(out + f".{r}.bf16.npy") for r in range(world)]
    np.testing.assert_array_equal(got[0], got[1])
    np.testing.assert_array_equal(gotb[0], gotb[1])
    # single process, the concatenated 2B batch, serial update
    net = _make_net(world * B)
    X, lab = _batch(0, world * B)
    net.a[0].copy_(torch.from_numpy(X).to(net.a[0].dtype))
    net.labels.copy_(torch.from_numpy(lab))
    for _ in range(2):
        net.step(overlap_update=False)
    torch.cuda.synchronize()
    ref = net.params.cpu().numpy()
    moved = np.abs(ref - _make_net(world * B).params.cpu().numpy())
    err = np.abs(got[0] - ref)
    # FP32 summation order (two half-batch sums vs one) is the only difference: far below the step
    assert err.max() <= 1e-3 * moved.max() + 1e-7, (err.max(), moved.max())
    assert np.sqrt(np.mean(err ** 2)) <= 1e-4 * np.sqrt(np.mean(moved ** 2))


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("graph", [False, True])
def test_dp_modes_single_rank_nccl(mode, graph):
    """World size 1 over NCCL: the exchange is the identity, so every mode -- eager, and captured
    with its collectives in one CUDA graph -- equals the serial step bit for bit."""
    import torch
    import torch.distributed as dist
    port = _free_port()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        outs = []
        for dp in (False, True):
            net = _make_net(16, seed=6)
            X, lab = _batch(0, 16)
            net.a[0].copy_(torch.from_numpy(X).to(net.a[0].dtype))
            net.labels.copy_(torch.from_numpy(lab))
            sync = _sync(mode, net, 1, 0) if dp else None
            if dp and graph:
                net.step(sync)                       # eager warm-up (workspaces, communicator)
                torch.cuda.synchronize()
                net.capture(allreduce=sync)
                net.graph.replay()
            else:
                for _ in range(2):
                    net.step(sync) if dp else net.step(overlap_update=False)
            torch.cuda.synchronize()
            outs.append((net.params.cpu().numpy().copy(), net.params_bf16.float().cpu().numpy().copy()))
        np.testing.assert_array_equal(outs[0][0], outs[1][0])
        np.testing.assert_array_equal(outs[0][1], outs[1][1])
    finally:
        dist.destroy_process_group()


def _guard_worker(rank, world, port, mode, out):
    import torch
    import torch.distributed as dist
    try:
        torch.cuda.set_device(0)
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1408_5093_b200.solver import Solver
        net = _make_net(B)
        X, lab = _batch(rank * B, B)
        net.a[0].copy_(torch.from_numpy(X).to(net.a[0].dtype))
        net.labels.copy_(torch.from_numpy(lab))
        sync = _sync(mode, net, world, rank)
        solver = Solver(torch.device("cuda", 0), "step", base_lr=0.05, gamma=0.5, stepsize=1)
        net.step(sync, solver=solver)
        torch.cuda.synchronize()
        before = net.params.cpu().numpy().copy()
        if rank == 1:
            net.labels[3] = 10                      # a corrupted label on ONE rank
        net.step(sync, solver=solver)
        torch.cuda.synchronize()
        st = solver.read()
        np.save(out + f".{rank}.npy", np.array([float(st["diverged"]), float(st["iter"]),
                                                 float(np.array_equal(before, net.params.cpu().numpy()))]))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback
        with open(out + f".{rank}.err", "w") as f:
            f.write(traceback.format_exc())


@pytest.mark.parametrize("mode", ["allreduce", "sharded"])
def test_dp_divergence_guard_is_global(tmp_path, mode):
    """With a solver, the data-parallel step averages the loss over the ranks before the guard
    (S:524): a non-finite loss on one rank makes EVERY rank skip the update (parameters unchanged
    everywhere, the iteration counter stopped), instead of the healthy ranks updating their slices
    with gradients that already carry the bad rank's NaNs."""
    import torch.multiprocessing as mp
    world = 2
    out = str(tmp_path / "g")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_guard_worker, args=(r, world, port, mode, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    for r in range(world):
        if os.path.exists(out + f".{r}.err"):
            pytest.fail(open(out + f".{r}.err").read())
        diverged, it, unchanged = np.load(out + f".{r}.npy")
        assert diverged == 1.0 and it == 1.0 and unchanged == 1.0, (r, diverged, it, unchanged)
