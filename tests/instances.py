"""Random problem builders shared by the tests (numpy RNG; the reference's
testutil.hpp:52-96 shapes and value ranges)."""
from __future__ import annotations

import numpy as np

from pyoracle import Problem, random_md


def int_instance(rng: np.random.Generator, with_exponents: bool, m: int = 1, cplx: bool = False,
                 nmax: int = 6, Nmax: int = 10, dmax: int = 5) -> Problem:
    """random_int_instance (testutil.hpp:52-72): n <= 6, N <= 10, d <= 5,
    coefficients in [1,9], inputs in [1,3], exponents in {1,2}; strictly
    positive, so the engine must equal the direct oracle bitwise."""
    n = int(rng.integers(1, nmax + 1))
    N = int(rng.integers(1, Nmax + 1))
    d = int(rng.integers(0, dmax + 1))
    nvars, idx, exps = [], [], []
    for _ in range(N):
        nk = int(rng.integers(1, min(n, 4) + 1))
        pick = sorted(rng.choice(np.arange(1, n + 1), nk, replace=False).tolist())
        nvars.append(nk)
        idx += pick
        if with_exponents and rng.integers(0, 2) == 1:
            exps += rng.integers(1, 3, nk).tolist()
        else:
            exps += [0] * nk
    P = 2 if cplx else 1
    top = 1 + N + n
    stat = np.zeros((P, m, top, d + 1))
    stat[:, 0, : 1 + N] = rng.integers(1, 10, (P, 1 + N, d + 1))
    stat[:, 0, 1 + N:] = rng.integers(1, 4, (P, n, d + 1))
    ex = np.array(exps, np.int32) if any(exps) else None
    return Problem(n, d, m, cplx, np.array(nvars, np.int32), np.array(idx, np.int32), ex, stat)


def md_instance(rng: np.random.Generator, m: int, cplx: bool = False, nmax: int = 6, Nmax: int = 8,
                dmax: int = 6, with_exponents: bool = False, dmin: int = 1) -> Problem:
    """random_md_instance (testutil.hpp:74-96): full-precision coefficients."""
    n = int(rng.integers(1, nmax + 1))
    N = int(rng.integers(1, Nmax + 1))
    d = int(rng.integers(dmin, dmax + 1))
    nvars, idx, exps = [], [], []
    for _ in range(N):
        nk = int(rng.integers(1, min(n, 4) + 1))
        pick = sorted(rng.choice(np.arange(1, n + 1), nk, replace=False).tolist())
        nvars.append(nk)
        idx += pick
        if with_exponents and rng.integers(0, 2) == 1:
            exps += rng.integers(1, 3, nk).tolist()
        else:
            exps += [0] * nk
    P = 2 if cplx else 1
    top = 1 + N + n
    vals = random_md(int(rng.integers(1, 2**62)), m, P * top * (d + 1))  # [count][m]
    stat = vals.reshape(P, top, d + 1, m).transpose(0, 3, 1, 2).copy()
    ex = np.array(exps, np.int32) if any(exps) else None
    return Problem(n, d, m, cplx, np.array(nvars, np.int32), np.array(idx, np.int32), ex, stat)


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def assert_bitwise(a, b, what=""):
    a, b = bits(a), bits(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    bad = np.argwhere(a != b)
    assert bad.size == 0, f"{what}: {len(bad)} mismatching words, first at {bad[:5].tolist()}"
