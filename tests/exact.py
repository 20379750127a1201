"""Exact-arithmetic references for pinning the oracle's floating point.

Correct rounding of an exact rational to IEEE binary32 (round to nearest,
ties to even), built from integer arithmetic only.  Used to check that the
oracle's ``fmaf`` steps are single-rounding fused multiply-adds (SURVEY.md
§8(c) O3 / pin P9) without trusting any float library.
"""
from fractions import Fraction

import numpy as np


def round_to_f32(q: Fraction) -> np.float32:
    if q == 0:
        return np.float32(0.0)
    sign = -1 if q < 0 else 1
    q = abs(q)
    e = q.numerator.bit_length() - q.denominator.bit_length() - 24
    while q / Fraction(2) ** e >= 2 ** 24:
        e += 1
    while q / Fraction(2) ** e < 2 ** 23 and e > -149:
        e -= 1
    e = max(e, -149)
    m = q / Fraction(2) ** e
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return np.float32(sign * float(fl) * 2.0 ** e)


def exact_fma_f32(a, x, y) -> np.float32:
    """round_f32(a*x + y) computed exactly (the definition of fmaf)."""
    q = Fraction(float(np.float32(a))) * Fraction(float(np.float32(x))) + Fraction(float(np.float32(y)))
    return round_to_f32(q)
