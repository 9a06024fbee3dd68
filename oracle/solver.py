"""Solver oracle -- TEST INFRASTRUCTURE ONLY (same import rules as the package).

PAPER.md P:171-178 (Sec. 3.4): "Caffe trains models by the fast and standard stochastic gradient
descent algorithm ... learning rate decay schedules, momentum, and snapshots".  The schedules and
the guard follow SPEC's solver module:
  * lr_at_iter   S:511-519  fixed / step / inv
  * sgd_step     S:520-528  zero diffs -> forward -> backward -> update; non-finite loss aborts
                 ("divergence guard", DESIGN DECISIONS S:570)
The update arithmetic itself is ``oracle.sgd_update`` (reading R18).
"""
from __future__ import annotations

import math

import numpy as np


class DivergenceError(RuntimeError):
    """a non-finite loss aborts the step before any parameter changes."""


def lr_at_iter(policy: str, base_lr: float, iter_: int, gamma: float = 0.0, stepsize: int = 1,
               power: float = 0.0) -> float:
    """fixed: base_lr; step: base_lr * gamma^floor(iter/stepsize);
    inv: base_lr * (1 + gamma*iter)^(-power).  fp64."""
    if iter_ < 0:
        raise ValueError("iter must be >= 0 (S:513)")
    if policy == "fixed":
        return float(base_lr)
    if policy == "step":
        return float(base_lr) * float(gamma) ** (iter_ // int(stepsize))
    if policy == "inv":
        return float(base_lr) * (1.0 + float(gamma) * iter_) ** (-float(power))
    raise ValueError(f"unknown lr policy {policy}")


def guarded_step(loss: float, params: dict, moms: dict, grads: dict, lr: float, momentum: float, decay: float,
                 grad_scale: float = 1.0):
    """S:523-524 one update of every parameter (w, v) -> oracle.sgd_update, unless the batch loss is
    non-finite: then DivergenceError is raised and nothing is modified."""
    import oracle
    if not math.isfinite(loss):
        raise DivergenceError(f"non-finite loss {loss}")
    for k in params:
        for t in range(len(params[k])):
            w, v = oracle.sgd_update(params[k][t], grads[k][t], moms[k][t], lr, momentum, decay, grad_scale)
            params[k][t][...] = w
            moms[k][t][...] = v
