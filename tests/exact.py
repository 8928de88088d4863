"""Exact rational arithmetic for accuracy envelopes (test infrastructure).

The reference checks its engine against an MPFR big-float oracle at
oracle_bits(m) = 64m+64 bits (bigreal.hpp:61, oracle_bigfloat.cpp); MPFR is
absent here. Multi-double values are finite sums of binary64 numbers, so
Python's Fraction represents every input exactly and series products and sums
of them exactly -- a stricter reference than any finite big-float precision.
"""
from __future__ import annotations

from fractions import Fraction
from typing import List, Sequence

import numpy as np

Series = List[Fraction]


def md_frac(limbs: Sequence[float]) -> Fraction:
    """Exact value of one multi-double (sum of its limbs)."""
    return sum((Fraction(float(v)) for v in limbs), Fraction(0))


def series_frac(s: np.ndarray) -> Series:
    """[m][d+1] limb-major series -> exact coefficients."""
    return [md_frac(s[:, k]) for k in range(s.shape[1])]


def conv(x: Series, y: Series) -> Series:
    d1 = len(x)
    return [sum((x[i] * y[k - i] for i in range(k + 1)), Fraction(0)) for k in range(d1)]


def add(x: Series, y: Series) -> Series:
    return [a + b for a, b in zip(x, y)]


def scale(x: Series, q: int) -> Series:
    return [a * q for a in x]


def power(x: Series, e: int) -> Series:
    out = [Fraction(1)] + [Fraction(0)] * (len(x) - 1)
    for _ in range(e):
        out = conv(out, x)
    return out


def evaluate_exact(p) -> tuple[Series, List[Series]]:
    """Value and gradient series of a real-mode Problem (pyoracle.Problem),
    exactly: f = a0 + sum_k a_k prod_j z_{i_j}^{e_j}, df/dz_i by the power
    rule, every product truncated at degree d (SPEC of evaluate)."""
    assert not p.cplx
    st = p.stat[0]  # [m][slots][d+1]
    a0 = series_frac(st[:, 0])
    z = [series_frac(st[:, 1 + p.N + i]) for i in range(p.n)]
    d1 = p.d + 1
    zero = [Fraction(0)] * d1
    value = list(a0)
    grad = [list(zero) for _ in range(p.n)]
    pos = 0
    for k in range(p.N):
        nk = int(p.nvars[k])
        idx = [int(v) - 1 for v in p.idx[pos:pos + nk]]
        ex = [1] * nk if p.exps is None else [max(1, int(v)) for v in p.exps[pos:pos + nk]]
        pos += nk
        a = series_frac(st[:, 1 + k])
        term = a
        for i, e in zip(idx, ex):
            term = conv(term, power(z[i], e))
        value = add(value, term)
        for j, (i, e) in enumerate(zip(idx, ex)):
            g = scale(a, e)
            for jj, (i2, e2) in enumerate(zip(idx, ex)):
                g = conv(g, power(z[i2], e2 - 1 if jj == j else e2))
            grad[i] = add(grad[i], g)
    return value, grad


def gap(md: Sequence[float], ref: Fraction) -> float:
    """|md - ref| as a double (underflow to 0 is fine, as in big_abs_gap)."""
    return abs(float(md_frac(md) - ref))


def rel_error(md: Sequence[float], ref: Fraction) -> float:
    """rel_error_vs (bigreal.cpp:14-26): |x - ref| / |ref|, or |x - ref| when
    ref is zero."""
    diff = abs(md_frac(md) - ref)
    return float(diff) if ref == 0 else float(diff / abs(ref))


def norm(s: Series) -> float:
    """big_norm (test_oracle.cpp:25-29): max |coefficient|, floored at 2^-300."""
    return max(max((abs(float(v)) for v in s), default=0.0), 2.0 ** -300)
