"""Shared helpers for the GPU parity tests (comparison metrics + device plumbing)."""
import numpy as np


def rel_l2(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref.ravel())
    return float(np.linalg.norm((got - ref).ravel()) / (den if den > 0 else 1.0))


def assert_fp32_close(got, ref, what=""):
    """BJ.north_star FP32-FMA bar: per element |err| <= 1e-5 * (|ref| + 1)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(got - ref)
    bound = 1e-5 * (np.abs(ref) + 1.0)
    bad = err > bound
    assert not bad.any(), f"{what}: {bad.sum()} / {bad.size} elements exceed 1e-5(|ref|+1); max err {err.max():.3e}"


def assert_tc_close(got, ref, what="", tol=1e-3):
    """BJ.north_star BF16/TF32 bar: relative L2 error <= 1e-3 vs the quantized-operand oracle."""
    e = rel_l2(got, ref)
    assert e <= tol, f"{what}: rel L2 {e:.3e} > {tol}"
    return e


def cuda(a, dtype=None):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.to(dtype) if dtype is not None else t


def host(t):
    import torch
    return t.detach().float().cpu().numpy() if t.dtype == torch.bfloat16 else t.detach().cpu().numpy()
