"""Accuracy envelopes and analytic identities, the reference's non-bitwise
checks (SURVEY.md 8(c) pin table), against an exact rational reference
(tests/exact.py) in place of the MPFR oracle:

  md add/mul relative error <= 2^(16-52m)        test_multidouble.cpp:185-205
  m = 1 is plain binary64                       test_multidouble.cpp:207-216
  Euler degree identity, exact on integers      test_executor.cpp:219-236
  Euler degree identity within the envelope     test_executor.cpp:238-269
  degree-0 finite difference == gradient        test_executor.cpp:271-290
  engine vs big-float at m=4, d=16              test_executor.cpp:292-310

The CPU tests hold the oracle to the envelope; the GPU tests hold the device
engine (through the C ABI) to the same bounds."""
import math

import numpy as np
import pytest

import exact
import pyoracle as po
from instances import int_instance, md_instance

LEVELS = [2, 3, 4, 5, 8, 10]


def md_rel_tolerance(m: int) -> float:
    return math.ldexp(1.0, 16 - 52 * m)  # multidouble.hpp:117


def worst_rel(x, y, s, p):
    wa = wm = 0.0
    for i in range(len(x)):
        fx, fy = exact.md_frac(x[i]), exact.md_frac(y[i])
        wa = max(wa, exact.rel_error(s[i], fx + fy))
        wm = max(wm, exact.rel_error(p[i], fx * fy))
    return wa, wm


@pytest.mark.parametrize("m", LEVELS)
def test_oracle_md_envelope(m):
    x = po.random_md(31 * m, m, 1500)
    y = po.random_md(31 * m + 1, m, 1500)
    wa, wm = worst_rel(x, y, po.md_op("add", x, y), po.md_op("mul", x, y))
    assert wa <= md_rel_tolerance(m) and wm <= md_rel_tolerance(m), (wa, wm)


def test_oracle_engine_vs_exact_m4_d16():
    rng = np.random.default_rng(511)
    p = md_instance(rng, 4, nmax=5, Nmax=6, dmax=16, dmin=16)
    vg = po.evaluate(p, "port")[0]  # [m][n+1][d+1]
    check_engine_vs_exact(p, vg)


def check_engine_vs_exact(p, vg):
    """tol = 2^(16-52m) * 64 * max|ref coefficient| per output series
    (test_executor.cpp:292-310)."""
    value, grad = exact.evaluate_exact(p)
    tol = md_rel_tolerance(p.m) * 64.0
    for s, ref in [(0, value)] + [(1 + i, g) for i, g in enumerate(grad)]:
        nrm = exact.norm(ref)
        for k in range(p.d + 1):
            assert exact.gap(vg[:, s, k], ref[k]) <= tol * nrm, (s, k)


# ---------------------------------------------------------------- device
pe = pytest.importorskip("paper_2101_10881_b200")


def dev_eval(p):
    st = p.stat.reshape(p.P * p.m, 1, *p.stat.shape[2:])
    vg, _ = pe.evaluate_packed(p.n, p.d, p.m, "real", p.nvars, p.idx, p.exps, st, 1)
    return vg[:, 0]  # [m][n+1][d+1]


@pytest.mark.gpu
@pytest.mark.parametrize("m", LEVELS)
def test_device_md_envelope(m):
    x = po.random_md(31 * m, m, 1500)
    y = po.random_md(31 * m + 1, m, 1500)
    wa, wm = worst_rel(x, y, pe.md_apply("add", x, y), pe.md_apply("mul", x, y))
    assert wa <= md_rel_tolerance(m) and wm <= md_rel_tolerance(m), (wa, wm)


@pytest.mark.gpu
def test_device_m1_is_binary64():
    rng = np.random.default_rng(55)
    a = rng.uniform(-1, 1, (5000, 1))
    b = rng.uniform(-1, 1, (5000, 1))
    assert (pe.md_apply("add", a, b) == a + b).all()
    assert (pe.md_apply("sub", a, b) == a - b).all()
    assert (pe.md_apply("mul", a, b) == a * b).all()


def single_monomial(p):
    """Keep the first monomial only and set a0 = 0 (homogeneous)."""
    nk = int(p.nvars[0])
    stat = p.stat[:, :, [0, 1] + list(range(1 + p.N, 1 + p.N + p.n))].copy()
    stat[:, :, 0] = 0.0
    ex = None if p.exps is None else p.exps[:nk].copy()
    q = po.Problem(p.n, p.d, p.m, p.cplx, p.nvars[:1].copy(), p.idx[:nk].copy(), ex, stat)
    deg = sum(1 if ex is None else max(1, int(e)) for e in (ex if ex is not None else [0] * nk))
    return q, deg


@pytest.mark.gpu
def test_device_euler_identity_exact_on_integers():
    """sum_i z_i * df/dz_i == deg * f for one monomial, exactly (integers)."""
    rng = np.random.default_rng(508)
    for it in range(30):
        p, deg = single_monomial(int_instance(rng, True))
        vg = dev_eval(p)
        z = [exact.series_frac(p.stat[0][:, 1 + p.N + i]) for i in range(p.n)]
        lhs = [0] * (p.d + 1)
        for i in range(p.n):
            lhs = exact.add(lhs, exact.conv(z[i], exact.series_frac(vg[:, 1 + i])))
        assert lhs == exact.scale(exact.series_frac(vg[:, 0]), deg), it


@pytest.mark.gpu
@pytest.mark.parametrize("m", [2, 4])
def test_device_euler_identity_within_envelope(m):
    rng = np.random.default_rng(509 + m)
    for it in range(10):
        p, deg = single_monomial(md_instance(rng, m, nmax=6, Nmax=2, dmax=5, with_exponents=True))
        vg = dev_eval(p)
        z = [exact.series_frac(p.stat[0][:, 1 + p.N + i]) for i in range(p.n)]
        lhs = [0] * (p.d + 1)
        termnorm = 0.0
        for i in range(p.n):
            t = exact.conv(z[i], exact.series_frac(vg[:, 1 + i]))
            termnorm = max(termnorm, max(abs(float(v)) for v in t))
            lhs = exact.add(lhs, t)
        rhs = exact.scale(exact.series_frac(vg[:, 0]), deg)
        tol = math.ldexp(1.0, 20 - 52 * m) * max(termnorm, 1.0)
        for k in range(p.d + 1):
            assert abs(float(lhs[k] - rhs[k])) <= tol, (it, k)


@pytest.mark.gpu
def test_device_finite_difference_matches_gradient():
    rng = np.random.default_rng(510)
    h = 2.0 ** -20
    for it in range(10):
        m = 2 + it % 2
        p = md_instance(rng, m)
        base = dev_eval(p)
        var = int(p.idx[0]) - 1
        q = po.Problem(p.n, p.d, p.m, p.cplx, p.nvars, p.idx, p.exps, p.stat.copy())
        slot = 1 + p.N + var
        hv = np.zeros((1, m))
        hv[0, 0] = h
        q.stat[0, :, slot, 0] = pe.md_apply("add", p.stat[0, :, slot, 0][None, :].copy(), hv)[0]
        pert = dev_eval(q)
        dv = float(exact.md_frac(pert[:, 0, 0]) - exact.md_frac(base[:, 0, 0])) / h
        gd = float(exact.md_frac(base[:, 1 + var, 0]))
        assert abs(dv - gd) <= 1e-6 * max(abs(gd), 1e-3), (it, dv, gd)


@pytest.mark.gpu
def test_device_engine_vs_exact_m4_d16():
    rng = np.random.default_rng(511)
    p = md_instance(rng, 4, nmax=5, Nmax=6, dmax=16, dmin=16)
    check_engine_vs_exact(p, dev_eval(p))


@pytest.mark.gpu
def test_device_engine_vs_exact_m10_d8():
    """the same envelope at the benchmark precision"""
    rng = np.random.default_rng(512)
    p = md_instance(rng, 10, nmax=4, Nmax=5, dmax=8, dmin=8)
    check_engine_vs_exact(p, dev_eval(p))
