"""Data-parallel gradient exchange.

The batch is sharded across ranks (per-image independence); the only exchange is the sum of
the parameter gradients.  Gradients live in ONE flat FP32 buffer laid out in forward order, so the
backward pass produces them from the end of the buffer towards the start.  Buckets are contiguous
ranges of that buffer, closed in backward order; as soon as the last layer of a bucket has enqueued
its weight gradient, an asynchronous ``all_reduce(SUM)`` of the bucket is issued (NCCL over
NVLink on the GPU; gloo in the CPU tests).  The collective is ordered after the gradient kernels on
the current stream and overlaps the rest of the backward pass; ``finish()`` makes the current
stream wait for every bucket.  The 1/W averaging is folded into the SGD update (reading R17).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple


class GradAllReduce:
    def __init__(self, flat_grads, segments: Sequence[Tuple[object, int, int]], world: int,
                 bucket_bytes: int = 32 << 20, group=None):
        """segments: (key, offset, numel) of every parameter tensor's gradient in `flat_grads`."""
        self.flat = flat_grads
        self.world = world
        self.group = group
        esz = flat_grads.element_size()
        segs = sorted(segments, key=lambda s: -s[1])          # backward order = descending offset
        self.buckets: List[Tuple[int, int, frozenset]] = []
        cur_keys, lo, hi, size = [], None, None, 0
        for key, off, n in segs:
            if not cur_keys:
                hi = off + n
            cur_keys.append(key)
            lo = off
            size += n * esz
            if size >= bucket_bytes:
                self.buckets.append((lo, hi, frozenset(cur_keys)))
                cur_keys, size = [], 0
        if cur_keys:
            self.buckets.append((0 if not self.buckets else lo, hi, frozenset(cur_keys)))
        # make the buckets tile [0, numel) exactly (alignment padding between tensors included)
        tiled, top = [], flat_grads.numel()
        for bi, (blo, bhi, keys) in enumerate(self.buckets):
            nlo = 0 if bi == len(self.buckets) - 1 else blo
            tiled.append((nlo, top, keys))
            top = nlo
        self.buckets = tiled
        self.key_bucket: Dict[object, int] = {}
        for bi, (_, _, keys) in enumerate(self.buckets):
            for k in keys:
                self.key_bucket[k] = bi
        self._pending = [set(b[2]) for b in self.buckets]
        self._works = []

    def reduce_loss(self, loss) -> None:
        """Replace this rank's loss (a device scalar) by the mean over the ranks, in place -- so a
        non-finite loss on any rank reaches every rank's divergence guard and all of them
        skip the same update."""
        import torch.distributed as dist
        if self.world <= 1:
            return
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(loss, op=dist.ReduceOp.AVG, group=self.group)
        else:
            dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=self.group)
            loss.div_(self.world)

    def on_grad(self, key) -> None:
        bi = self.key_bucket[key]
        p = self._pending[bi]
        p.discard(key)
        if not p:
            import torch.distributed as dist
            lo, hi, _ = self.buckets[bi]
            self._works.append(dist.all_reduce(self.flat[lo:hi], op=dist.ReduceOp.SUM, group=self.group,
                                               async_op=True))

    def finish(self) -> None:
        for w in self._works:
            w.wait()
        self._works = []
        self._pending = [set(b[2]) for b in self.buckets]


class BucketedSGD:
    """Data-parallel gradient exchange WITH the update, per bucket:

    mode "allreduce": as soon as a bucket's gradients are complete, ``all_reduce(SUM)`` it; as soon as
        its layers are also done with their weights (their data gradients have run), update the whole
        bucket (grad_scale = 1/W, reading R17) -- the update overlaps the rest of the backward pass
        instead of following it.
    mode "sharded" (reduce-scatter + sharded SGD + all-gather): ``reduce_scatter`` the bucket so that
        rank r receives the summed gradient of its 1/W slice, apply the update to that slice only (the
        update's 22 bytes/parameter of HBM traffic drop W-fold), then ``all_gather`` the updated FP32
        weights and their BF16 copy.  NCCL's in-place forms are used (each rank's slice is a view of
        the flat buffers), so no staging copies exist.

    The caller provides ``update(lo, hi, grad_scale)`` (the library SGD on the flat range) and calls
    ``on_grad(key)`` when a layer's parameter gradients are enqueued, ``on_done(key)`` when nothing
    later in the step reads that layer's parameters, and ``finish()`` at the end of the backward
    pass (it makes the current stream wait for the last collectives).  Streams: collectives and
    updates are issued on ``stream`` (a side stream) after it waits for the producing stream.
    """

    applies_update = True     # Net.step: the exchange applies the SGD update itself

    def __init__(self, flat_grads, flat_params, flat_mom, flat_bf16, segments, world, rank, update=None, mode="sharded",
                 bucket_bytes=32 << 20, group=None, stream=None):
        import torch
        self.torch = torch
        self.mode = mode
        self.world, self.rank, self.group = world, rank, group
        self.update = update
        self.grads, self.params, self.mom, self.bf16 = flat_grads, flat_params, flat_mom, flat_bf16
        self.stream = stream
        self.cuda = flat_grads.is_cuda
        base = GradAllReduce(flat_grads, segments, world, bucket_bytes=bucket_bytes, group=group)
        self.buckets = base.buckets
        self.key_bucket = base.key_bucket
        if mode == "sharded":
            for lo, hi, _ in self.buckets:
                n = hi - lo
                # equal 16-byte-aligned slices per rank (the flat buffer keeps every tensor 256-byte aligned)
                if n % (4 * world) or (lo % 4):
                    raise ValueError(f"bucket [{lo},{hi}) does not split into {world} aligned slices")
        self._reset()

    reduce_loss = GradAllReduce.reduce_loss

    def _reset(self):
        self._grad_pending = [set(b[2]) for b in self.buckets]
        self._done_pending = [set(b[2]) for b in self.buckets]
        self._rs = {}
        self._tail = []

    def _slice(self, bi):
        lo, hi, _ = self.buckets[bi]
        if self.mode != "sharded":
            return lo, hi
        n = (hi - lo) // self.world
        return lo + self.rank * n, lo + (self.rank + 1) * n

    def _ctx(self):
        import contextlib
        if self.cuda and self.stream is not None:
            return self.torch.cuda.stream(self.stream)
        return contextlib.nullcontext()

    def _join_current(self):
        """The side stream waits for everything enqueued so far on the current stream."""
        if self.cuda and self.stream is not None:
            self.stream.wait_stream(self.torch.cuda.current_stream())

    def on_grad(self, key):
        import torch.distributed as dist
        bi = self.key_bucket[key]
        p = self._grad_pending[bi]
        p.discard(key)
        if p:
            return
        lo, hi, _ = self.buckets[bi]
        self._join_current()
        with self._ctx():
            if self.mode == "sharded":
                slo, shi = self._slice(bi)
                self._rs[bi] = dist.reduce_scatter_tensor(self.grads[slo:shi], self.grads[lo:hi], op=dist.ReduceOp.SUM,
                                                          group=self.group, async_op=True)
            else:
                self._rs[bi] = dist.all_reduce(self.grads[lo:hi], op=dist.ReduceOp.SUM, group=self.group,
                                               async_op=True)
        self._maybe_update(bi)

    def on_done(self, key):
        bi = self.key_bucket[key]
        self._done_pending[bi].discard(key)
        self._maybe_update(bi)

    def _maybe_update(self, bi):
        import torch.distributed as dist
        if self._done_pending[bi] or bi not in self._rs or self._rs[bi] is None:
            return
        work = self._rs[bi]
        self._rs[bi] = None
        self._join_current()          # after the data gradients that read this bucket's weights
        with self._ctx():
            work.wait()               # the reduced gradient slice (stream-ordered on CUDA)
            slo, shi = self._slice(bi)
            self.update(slo, shi, 1.0 / self.world)
            if self.mode == "sharded" and self.world > 1:
                lo, hi, _ = self.buckets[bi]
                self._tail.append(dist.all_gather_into_tensor(self.params[lo:hi], self.params[slo:shi],
                                                              group=self.group, async_op=True))
                if self.bf16 is not None:
                    self._tail.append(dist.all_gather_into_tensor(self.bf16[lo:hi], self.bf16[slo:shi],
                                                                  group=self.group, async_op=True))

    def finish(self):
        for bi in range(len(self.buckets)):
            if self._rs.get(bi) is not None or self._done_pending[bi]:
                raise RuntimeError(f"bucket {bi} was not completed by the backward pass")
        for w in self._tail:
            w.wait()
        if self.cuda and self.stream is not None:
            self.torch.cuda.current_stream().wait_stream(self.stream)
        self._reset()
