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


def bf16_ulp(x):
    """Spacing of BF16 values at |x| (8 significant bits): 2^(floor(log2|x|) - 7); the subnormal
    spacing 2^-133 below the normal range."""
    a = np.abs(np.asarray(x, np.float64))
    e = np.floor(np.log2(np.maximum(a, 2.0 ** -126)))
    return 2.0 ** (e - 7)


def bf16_ulp_errors(got, ref):
    """|got - RNE_bf16(ref)| in units of the BF16 spacing at RNE_bf16(ref) (per element)."""
    import oracle
    r = oracle.quant_bf16(np.asarray(ref, np.float32)).astype(np.float64)
    return np.abs(np.asarray(got, np.float64) - r) / bf16_ulp(r)


def assert_bf16_ulp(got, ref, what="", ulps=1.0, atol=0.0):
    """BF16-stored result within `ulps` BF16 spacings of RNE(oracle) per element (reading R12 for BF16
    outputs).  `atol` (absolute) admits FP32 accumulation error where the exact result cancels to
    ~0 (a tiny |ref| has a tiny spacing, the rounding of the long FP32 sum does not)."""
    import oracle
    got = np.asarray(got, np.float64)
    r = oracle.quant_bf16(np.asarray(ref, np.float32)).astype(np.float64)
    err = np.abs(got - r)
    bound = ulps * bf16_ulp(r) + atol
    bad = err > bound
    assert not bad.any(), (f"{what}: {int(bad.sum())} / {bad.size} elements beyond {ulps} BF16 ulp of RNE(ref)"
                           f" (+{atol:.2e}); worst err {err[bad].max():.3e} at ref {r[bad][np.argmax(err[bad])]:.3e}")
    return float((err / bf16_ulp(r)).max())
