"""Host checks of the arithmetic facts the CUDA kernels rely on (no GPU).

The channels-last max-pool backward (csrc/simple.cu, pool_block_k3s2) sums the two window
gradients that can reach an edge position of a 2x2 block with one packed BF16 add instead of
R8's FP32 sum followed by one BF16 rounding.  That is only bit-exact if
RN_bf16(RN_fp32(a + b)) == RN_bf16(a + b) for every pair of BF16 values; this test checks it
against exact rational arithmetic on a sample that sweeps the exponent gap across the point
(about 16 binades) where a + b stops being exact in FP32, with both signs and ties.
"""
from fractions import Fraction

import numpy as np
import pytest


def _bf16_values(bits):
    return (np.asarray(bits, dtype=np.uint32) << 16).view(np.float32)


def _rn_bf16_exact(q: Fraction) -> Fraction:
    """Round an exact rational to the nearest BF16 (8 significant bits), ties to even; normal range."""
    if q == 0:
        return Fraction(0)
    s = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    ulp = Fraction(2) ** (e - 7)
    m = a / ulp
    lo = m.numerator // m.denominator
    rem = m - lo
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and lo % 2 == 1):
        lo += 1
    return s * lo * ulp


def _rn_bf16_from_f32(x):
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)


@pytest.mark.parametrize("seed", [0, 1])
def test_two_term_bf16_sum_has_no_double_rounding(seed):
    rng = np.random.default_rng(seed)
    n = 4000
    exp_a = rng.integers(100, 150, n)
    gap = rng.integers(0, 30, n)
    exp_b = exp_a - gap
    man_a, man_b = rng.integers(0, 128, n), rng.integers(0, 128, n)
    sa, sb = rng.integers(0, 2, n), rng.integers(0, 2, n)
    a = _bf16_values((sa << 15) | (exp_a << 7) | man_a)
    b = _bf16_values((sb << 15) | (exp_b << 7) | man_b)
    via_f32 = _rn_bf16_from_f32(np.float32(a) + np.float32(b))
    for i in range(n):
        exact = _rn_bf16_exact(Fraction(float(a[i])) + Fraction(float(b[i])))
        assert Fraction(float(via_f32[i])) == exact, (float(a[i]), float(b[i]))
