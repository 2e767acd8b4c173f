"""Third, independent implementation of Eq. 1 in exact rational arithmetic
(``fractions.Fraction``), used only to pin the oracle.

It shares nothing with oracle/ beyond reading the same rules S1-S4 from the
paper's Eq. 1: every rounding here is computed exactly.
"""

from __future__ import annotations

from fractions import Fraction

F16_MAX = Fraction(65504)
F16_QUANTUM_MIN = Fraction(1, 2 ** 24)


def _quantum_f16(x: Fraction) -> Fraction:
    """Spacing of fp16 values in the binade containing |x| (x > 0)."""
    e = 0
    a = abs(x)
    # find e with 2^e <= a < 2^(e+1)
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    if e < -14:
        return F16_QUANTUM_MIN
    return Fraction(2) ** (e - 10)


def rz_f16(x: Fraction) -> Fraction:
    """Exact round-toward-zero to fp16 (saturating at 65504)."""
    if x == 0:
        return Fraction(0)
    s = 1 if x > 0 else -1
    a = abs(x)
    if a >= F16_MAX:
        return s * F16_MAX
    q = _quantum_f16(a)
    return s * (a // q) * q


def rn_f16(x: Fraction) -> Fraction:
    """Exact round-to-nearest-even to fp16 (Inf as None when it overflows)."""
    if x == 0:
        return Fraction(0)
    s = 1 if x > 0 else -1
    a = abs(x)
    q = _quantum_f16(a)
    lo = (a // q) * q
    rem = a - lo
    if rem * 2 > q:
        r = lo + q
    elif rem * 2 < q:
        r = lo
    else:
        r = lo if ((lo / q) % 2 == 0) else lo + q
    if r > F16_MAX:
        # overflow threshold: values >= 65520 round to Inf
        return None
    return s * r


def rha(x: Fraction) -> int:
    """Exact round half away from zero."""
    n = (abs(x) + Fraction(1, 2)).__floor__()
    return n if x >= 0 else -n


def quantize_group(values, n_bits: int = 4):
    """Eq. 1 with readings S1-S4, exactly.  values: fp16-representable floats.
    Returns (codes, delta (Fraction), Z (int))."""
    qmax = 2 ** n_bits - 1
    F = [Fraction(v) for v in values]
    lo, hi = min(F), max(F)
    r = hi - lo
    if r > 0:
        d = rz_f16(r / qmax)
        if d == 0:
            d = F16_QUANTUM_MIN
    else:
        d = Fraction(1) if lo == 0 else abs(lo)
    Z = min(max(rha(-lo / d), 0), qmax)
    codes = [min(max(rha(v / d) + Z, 0), qmax) for v in F]
    return codes, d, Z


# bfloat16: 8-bit significand (7 stored bits), fp32's exponent range (emin = -126,
# subnormal quantum 2^-133), largest finite (2 - 2^-7) * 2^127.
BF16_MAX = (2 - Fraction(1, 2 ** 7)) * Fraction(2) ** 127
BF16_QUANTUM_MIN = Fraction(1, 2 ** 133)


def _quantum_bf16(a: Fraction) -> Fraction:
    """Spacing of bf16 values in the binade containing a > 0."""
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    elif Fraction(2) ** (e + 1) <= a:
        e += 1
    if e < -126:
        return BF16_QUANTUM_MIN
    return Fraction(2) ** (e - 7)


def rn_bf16(x: Fraction):
    """Exact round-to-nearest-even to bf16; returns the value, or None on overflow
    (|x| at or above the midpoint between BF16_MAX and 2^128 rounds to Inf)."""
    if x == 0:
        return Fraction(0)
    s = 1 if x > 0 else -1
    a = abs(x)
    q = _quantum_bf16(a)
    lo = (a // q) * q
    rem = a - lo
    if rem * 2 > q:
        r = lo + q
    elif rem * 2 < q:
        r = lo
    else:
        r = lo if ((lo / q) % 2 == 0) else lo + q
    if r > BF16_MAX:
        return None
    return s * r
