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
