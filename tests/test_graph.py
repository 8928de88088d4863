"""Host side of the product (C++ graph compiler, generator, cost model) --
CPU only. Known answers from the reference tests (test_jobgraph.cpp,
acceptance.cpp criteria 1-4, test_executor.cpp:312-345) and job-for-job
equality with the oracle's build_jobgraph."""
import json
import os

import numpy as np
import pytest

import paper_2101_10881_b200 as pe
import pyoracle as po
from instances import assert_bitwise

GOLD = os.path.join(os.path.dirname(__file__), "golden")
META = json.load(open(os.path.join(GOLD, "golden.json")))


def rows(g):
    conv = np.stack([np.repeat(np.arange(1, len(g.conv_layer_off)), np.diff(g.conv_layer_off)), g.conv_in1,
                     g.conv_in2, g.conv_out, g.conv_copy.astype(np.int64)], 1)
    add = np.stack([np.repeat(np.arange(1, len(g.add_layer_off)), np.diff(g.add_layer_off)), g.add_src, g.add_dst], 1)
    return conv, add


def same_as_oracle(g, p: po.Problem):
    o = po.graph(p, "port")
    conv, add = rows(g)
    assert g.total_slots == o["total_slots"]
    assert (conv == o["conv"]).all()
    assert (add == o["add"]).all()
    assert g.value_slot == o["value_slot"]
    assert (g.gradient_slots == o["grad_slots"]).all()
    assert (g.multipliers == o["mult"]).all()
    assert (g.term_scales.reshape(-1, 2) == o["term_scales"].reshape(-1, 2)).all()


def shape_problem(n, d, monos, exps=None):
    nv = np.array([len(x) for x in monos], np.int32)
    idx = np.array([i for x in monos for i in x], np.int32)
    ex = None if exps is None else np.array([e for x in exps for e in x], np.int32)
    return po.Problem(n, d, 1, False, nv, idx, ex, None)


@pytest.mark.parametrize("pid", ["p1", "p2", "p3"])
def test_benchmark_graphs_equal_oracle(pid):
    pr = pe.gen_benchmark(pid, 4, 1, with_static=False)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    same_as_oracle(g, po.Problem(pr.n, 4, 1, False, pr.nvars, pr.indices, None, None))
    want = META["graphs"][pid]
    assert g.conv_layer_sizes() == want["conv_layers"] and g.add_layer_sizes() == want["add_layers"]
    assert pe.validate(g) == (True, "")


def test_acceptance_counts():
    """acceptance.cpp criteria 1 and 3, test_jobgraph.cpp:216-245."""
    g1 = pe.build_jobgraph_shape(16, 8, *pe_shape("p1"))
    assert g1.conv_job_count() == 16380 and g1.add_job_count() == 9084
    assert g1.conv_layer_sizes() == [3640, 5460, 5460, 1820]
    assert g1.add_layer_sizes() == [4542, 2279, 1140, 562, 281, 140, 78, 39, 20, 2, 1]
    g2 = pe.build_jobgraph_shape(128, 4, *pe_shape("p2"))
    assert g2.conv_job_count() == 24192 and g2.add_job_count() == 8192 and len(g2.add_layer_sizes()) == 8
    g3 = pe.build_jobgraph_shape(128, 4, *pe_shape("p3"))
    assert g3.conv_job_count() == 24384 and g3.add_job_count() == 24256
    # 455 terms per variable in p1 (C(15,3)): the gradient lists
    per_var = np.bincount(pe_shape("p1")[1])[1:]
    assert (per_var == 455).all()


def pe_shape(pid):
    pr = pe.gen_benchmark(pid, 1, 1, with_static=False)
    return pr.nvars, pr.indices


def test_worked_example():
    """x1x3x6 + x1x2x5x6 + x2x3x4 (test_jobgraph.cpp:46-71, acceptance criterion 2)."""
    d = 2
    g = pe.build_jobgraph_shape(6, d, [3, 4, 3], [1, 3, 6, 1, 2, 5, 6, 2, 3, 4])
    assert g.total_slots == 28
    assert g.conv_job_count() == 21 and g.conv_layer_sizes() == [6, 9, 5, 1]
    first = [j for j in g.conv_layers[0] if j[2] == 10][0]  # f_{0,1}
    assert (first[0] * (d + 1), first[1] * (d + 1), first[2] * (d + 1)) == (d + 1, 4 * d + 4, 10 * d + 10)
    src, dst, _ = g.add_layers[0][0]
    assert (src * (d + 1), dst * (d + 1)) == (0, 12 * d + 12)


def test_single_monomial_job_lists():
    """per-n_k job lists (test_jobgraph.cpp:79-110)."""
    g = pe.build_jobgraph_shape(1, 1, [1], [1])
    assert g.conv_job_count() == 2 and g.copy_job_count() == 1
    g = pe.build_jobgraph_shape(2, 1, [2], [1, 2])
    assert [len(L) for L in g.conv_layers] == [2, 1]
    for nk in (3, 4, 5, 7):
        g = pe.build_jobgraph_shape(nk, 1, [nk], list(range(1, nk + 1)))
        assert g.conv_job_count() == 3 * nk - 3 and len(g.conv_layer_sizes()) == nk


def test_random_shapes_equal_oracle():
    rng = np.random.default_rng(1234)
    for it in range(300):
        n = int(rng.integers(1, 12))
        N = int(rng.integers(1, 15))
        monos, exps = [], []
        for _ in range(N):
            nk = int(rng.integers(1, min(n, 7) + 1))
            monos.append(sorted(rng.choice(np.arange(1, n + 1), nk, replace=False).tolist()))
            exps.append(rng.integers(1, 4, nk).tolist() if rng.integers(0, 3) == 0 else [0] * nk)
        has = any(any(e) for e in exps)
        p = shape_problem(n, 3, monos, exps if has else None)
        g = pe.build_jobgraph_shape(n, 3, p.nvars, p.idx, p.exps)
        same_as_oracle(g, p)
        ok, msg = pe.validate(g)
        assert ok, msg


def test_injected_violations_are_rejected():
    """test_jobgraph.cpp:331-362: a job moved one layer early, a duplicate write."""
    g = pe.build_jobgraph_shape(16, 2, *pe_shape("p1"))
    base = pe.GraphArrays.from_graph(g)
    assert pe.validate(base) == (True, "")
    # move the first layer-2 job into layer 1: it now reads a slot not yet written
    off = g.conv_layer_off.copy()
    off[1] += 1
    bad = pe.GraphArrays(g.n, g.N, g.d, g.total_slots, g.value_slot, g.gradient_slots, g.multipliers, off,
                         g.conv_in1, g.conv_in2, g.conv_out, g.conv_copy, g.add_layer_off, g.add_src, g.add_dst)
    ok, msg = pe.validate(bad)
    assert not ok and "not written in an earlier layer" in msg
    # duplicate write inside one layer
    out = g.conv_out.copy()
    out[1] = out[0]
    bad = pe.GraphArrays(g.n, g.N, g.d, g.total_slots, g.value_slot, g.gradient_slots, g.multipliers,
                         g.conv_layer_off, g.conv_in1, g.conv_in2, out, g.conv_copy, g.add_layer_off, g.add_src,
                         g.add_dst)
    ok, msg = pe.validate(bad)
    assert not ok and "duplicate write" in msg


def test_flop_totals():
    """test_executor.cpp:312-319 / acceptance criterion 4 / PAPER.md:918-923."""
    g = pe.build_jobgraph_shape(16, 8, *pe_shape("p1"))
    deca = pe.OpCost(397, 3089)
    assert pe.flop_count_mul(g, 152, "real", deca) == 1_184_444_368_380
    assert pe.flop_count_add(g, 152, "real", deca) == 151_782_283_404
    assert pe.flop_count(g, 152, "real", deca) == 1_336_226_651_784


def test_flop_small_cases():
    """test_executor.cpp:321-345."""
    unit = pe.OpCost(1, 1)
    # one conv job (slots 1,2 -> 3), n=1, N=1
    ga = pe.GraphArrays(1, 1, 0, 4, 3, [3], [1], [0, 1], [1], [2], [3], [0], [0], [], [])
    assert pe.flop_count(ga, 0, "real", unit) == 1
    assert pe.flop_count(ga, 1, "real", unit) == 6
    assert pe.flop_count_mul(ga, 1, "cplx", unit) == 16
    assert pe.flop_count_add(ga, 1, "cplx", unit) == 12
    ga = pe.GraphArrays(1, 1, 0, 4, 3, [3], [1], [0, 2], [1, 1], [2, 0], [3, 2], [0, 1], [0, 1], [3], [2])
    assert pe.flop_count(ga, 1, "real", unit) == 8
    assert pe.flop_count_add(ga, 1, "cplx", unit) == 16


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 8, 10])
def test_cost_tables_pinned_to_reference(m):
    ia, im, ra, rm = META["costs"][str(m)]
    assert (pe.instrumented_cost(m).add_cost, pe.instrumented_cost(m).mul_cost) == (ia, im)
    assert (pe.reporting_cost(m).add_cost, pe.reporting_cost(m).mul_cost) == (ra, rm)


def test_unsupported_precision_is_invalid_argument():
    with pytest.raises(pe.InvalidArgument):
        pe.instrumented_cost(7)


@pytest.mark.parametrize("pid,d,m,mode", [("p1", 4, 10, "real"), ("p2", 2, 3, "real"), ("p3", 2, 2, "cplx"),
                                          ("p1", 7, 8, "cplx")])
def test_generator_bitwise_equal_oracle(pid, d, m, mode):
    a = pe.gen_benchmark(pid, d, m, mode, seed=7)
    b = po.gen_benchmark(pid, d, m, mode == "cplx", seed=7)
    assert (a.nvars == b.nvars).all() and (a.indices == b.idx).all()
    assert_bitwise(a.stat, b.stat.reshape(a.stat.shape), f"{pid} static block")


@pytest.mark.parametrize("bad", [
    dict(n=0, nvars=[1], idx=[1]),
    dict(n=3, nvars=[2], idx=[2, 1]),       # not increasing
    dict(n=3, nvars=[2], idx=[1, 4]),       # out of range
    dict(n=3, nvars=[0], idx=[]),           # no variables
])
def test_invalid_polynomials_rejected(bad):
    with pytest.raises(pe.InvalidArgument):
        pe.build_jobgraph_shape(bad["n"], 2, bad["nvars"], bad["idx"])


def test_negative_exponent_rejected():
    with pytest.raises(pe.InvalidArgument):
        pe.build_jobgraph_shape(2, 2, [2], [1, 2], [1, -1])


def test_stage_layout_and_checks():
    """staging fills the static region, zeroes the dynamic one
    (test_executor.cpp:49-91)."""
    rng = np.random.default_rng(501)
    d, m = 1, 2
    ser = lambda: po.random_md(int(rng.integers(1, 2**40)), m, d + 1).T.reshape(1, m, d + 1).copy()
    mons = [pe.Monomial(ser(), ix) for ix in ([1, 3, 6], [1, 2, 5, 6], [2, 3, 4])]
    p = pe.Polynomial(6, d, ser(), mons)
    z = [ser() for _ in range(6)]
    a = pe.stage(p, z)
    assert a.total_slots == 28 and a.slabs.shape == (2, 28, 2)
    assert pe.series_bitwise_equal(a.read_slot(0), p.a0)
    assert pe.series_bitwise_equal(a.read_slot(3), mons[2].coeff)
    assert pe.series_bitwise_equal(a.read_slot(4), z[0])
    assert (a.slabs[:, 10:] == 0).all()
    with pytest.raises(pe.InvalidArgument):
        pe.stage(p, z[:-1])
    mons[0].exponents = [2, 1, 1]
    with pytest.raises(pe.InvalidArgument):
        pe.stage(p, z)
