"""Seeded synthetic inputs shared by the tests, the bench and smoke().

This module holds ONLY random draws (no arithmetic of the method): it is the one
module both the oracle-side tests and the CUDA path are fed from.  Every stream
is numpy PCG64 seeded with ``SeedSequence([seed, stream_id])`` so that a given
(seed, stream) pair always yields the same array regardless of call order.

Recipes:
  * per-layer parity: X, dY ~ U(-1, 1); W ~ xavier U(+-sqrt(3/fan_in));
    b ~ U(-1, 1)
  * LeNet: pixels round(U[0,255])/256 (S:589 scale), xavier weights
  * CaffeNet: mean-subtracted pixel surrogate = integers U{-128..127} (exact in
    bf16); conv/fc8 weights N(0, 0.01^2), fc6/fc7 N(0, 0.005^2); biases 0 or 1
  * labels U{0..K-1}
"""
from __future__ import annotations

import numpy as np

# stream ids (fixed order: [X, W, b, dY, labels])
S_X, S_W, S_B, S_DY, S_LABELS, S_AUX = 0, 1, 2, 3, 4, 5


def gen(seed: int, stream: int, sub: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), int(stream), int(sub)])))


def uniform(shape, seed, stream, sub=0, lo=-1.0, hi=1.0):
    return gen(seed, stream, sub).uniform(lo, hi, size=shape).astype(np.float32)


def xavier(shape, seed, stream=S_W, sub=0):
    fan_in = int(np.prod(shape[1:]))
    a = np.sqrt(3.0 / fan_in)
    return gen(seed, stream, sub).uniform(-a, a, size=shape).astype(np.float32)


def gaussian(shape, std, seed, stream=S_W, sub=0):
    return (gen(seed, stream, sub).standard_normal(size=shape) * std).astype(np.float32)


def int_pixels(shape, seed, stream=S_X, sub=0, lo=-128, hi=127):
    return gen(seed, stream, sub).integers(lo, hi + 1, size=shape).astype(np.float32)


def mnist_pixels(shape, seed, stream=S_X, sub=0):
    return (np.round(gen(seed, stream, sub).uniform(0, 255, size=shape)) / 256.0).astype(np.float32)


def labels(n, k, seed, stream=S_LABELS, sub=0):
    return gen(seed, stream, sub).integers(0, k, size=(n,)).astype(np.int32)


def distinct_values(shape, seed, spacing=0.01, stream=S_AUX, sub=0):
    """A random permutation of evenly spaced values: no ties, neighbours >= spacing apart
    (used for finite-difference checks away from max/ReLU kinks)."""
    n = int(np.prod(shape))
    v = (np.arange(n) - n / 2.0) * spacing
    return gen(seed, stream, sub).permutation(v).reshape(shape).astype(np.float64)


def class_pattern_pixels(labels, shape_chw, k, seed, noise=64.0, stream=S_AUX, sub=11):
    """Learnable synthetic images for a training-loop sanity run: one random template per class
    (integers U{0..255}) plus per-image integer noise U{-noise..noise}, clipped to [0, 255] and
    scaled by 1/256 (the LeNet input scale).  Only random draws and a clip -- no arithmetic
    of the method."""
    g = gen(seed, stream, sub)
    templates = g.integers(0, 256, size=(k,) + tuple(shape_chw))
    lab = np.asarray(labels).astype(np.int64)
    noise_v = g.integers(-int(noise), int(noise) + 1, size=(lab.shape[0],) + tuple(shape_chw))
    img = np.clip(templates[lab] + noise_v, 0, 255)
    return (img / 256.0).astype(np.float32)
