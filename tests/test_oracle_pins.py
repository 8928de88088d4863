"""Pin the CPU oracle (the plain-C restatement in oracle/pse_oracle.c) before
trusting it: against the golden vectors generated from the reference engine
itself (tests/golden/, by make_golden.py), and -- where the reference library
oracle/_ref was built -- against that library directly."""
import glob
import json
import os

import numpy as np
import pytest

import pyoracle as po
from instances import assert_bitwise, int_instance, md_instance

GOLD = os.path.join(os.path.dirname(__file__), "golden")
META = json.load(open(os.path.join(GOLD, "golden.json")))
LEVELS = [1, 2, 3, 4, 5, 8, 10]
needs_ref = pytest.mark.skipif(not po.has_ref(), reason="oracle/_ref not built (no /root/reference here)")


def load_problem(path):
    z = np.load(path)
    exps = z["exps"] if z["exps"].size else None
    p = po.Problem(int(z["n"]), int(z["d"]), int(z["m"]), bool(z["cplx"]), z["nvars"], z["idx"], exps, z["stat"])
    return p, z


@pytest.mark.parametrize("m", LEVELS)
def test_md_ops_match_golden(m):
    z = np.load(os.path.join(GOLD, f"md_m{m}.npz"))
    for op in ("add", "sub", "mul"):
        assert_bitwise(po.md_op(op, z["x"], z["y"]), z[op], f"{op} m={m}")


def test_rng_and_seed_mixing_match_golden():
    assert [int(v) for v in po.rng_u64(7, 8)] == META["rng_u64_seed7"]
    assert po.mix_seed(7, 1 << 32) == META["mix_seed_7_1<<32"]


@pytest.mark.parametrize("m", LEVELS)
def test_cost_tables_match_golden(m):
    assert list(po.cost(m)) == META["costs"][str(m)]


@pytest.mark.parametrize("pid", ["p1", "p2", "p3"])
def test_graph_shapes_match_golden(pid):
    g = po.graph(po.gen_benchmark(pid, 2, 1), "port")
    want = META["graphs"][pid]
    assert g["total_slots"] == want["total_slots"]
    assert len(g["conv"]) == want["conv"] and len(g["add"]) == want["add"]
    assert np.bincount(g["conv"][:, 0])[1:].tolist() == want["conv_layers"]
    assert np.bincount(g["add"][:, 0])[1:].tolist() == want["add_layers"]
    assert int(np.bitwise_xor.reduce((g["conv"] * np.arange(1, len(g["conv"]) + 1)[:, None]).ravel())) == want["conv_sha"]
    assert int(np.bitwise_xor.reduce((g["add"] * np.arange(1, len(g["add"]) + 1)[:, None]).ravel())) == want["add_sha"]
    assert g["valid"], g["message"]


def test_flop_totals_match_golden_and_paper():
    p1 = po.gen_benchmark("p1", 2, 1)
    got = [po.flop_count(p1, 397, 3089, w, d=152) for w in (0, 1, 2)]
    assert got == META["flops_p1_d152_deca"]
    # the paper's published totals (test_executor.cpp:312-319)
    assert got == [1_336_226_651_784, 1_184_444_368_380, 151_782_283_404]


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "vg_*.npy"))), ids=os.path.basename)
def test_engine_outputs_match_golden(path):
    name = os.path.basename(path)[3:-4].split("_")
    pid, d, m = name[0], int(name[1][1:]), int(name[2][1:])
    cplx = len(name) > 3
    p = po.gen_benchmark(pid, d, m, cplx, seed=7)
    assert_bitwise(po.evaluate(p, "port"), np.load(path), name)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "int_*.npz"))), ids=os.path.basename)
def test_integer_instances_match_golden(path):
    p, z = load_problem(path)
    assert_bitwise(po.evaluate(p, "port"), z["vg"], "engine")
    assert_bitwise(po.eval_direct(p, "port"), z["direct"], "direct")
    # positive integers: the graph engine equals the direct oracle bitwise
    assert_bitwise(z["vg"], z["direct"], "engine vs direct")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "md_[0-9]*.npz"))), ids=os.path.basename)
def test_md_instances_match_golden(path):
    p, z = load_problem(path)
    assert_bitwise(po.evaluate(p, "port"), z["vg"], os.path.basename(path))


def test_random_md_generation_is_normalized_and_deterministic():
    for m in LEVELS:
        a = po.random_md(5, m, 100)
        assert_bitwise(a, po.random_md(5, m, 100))
        assert (np.abs(a[:, 0]) <= 1.0).all()


# --------------------------------------------------- direct reference pins
@needs_ref
@pytest.mark.parametrize("m", LEVELS)
def test_md_ops_match_reference_library(m):
    x = po.random_md(900 + m, m, 20000, "ref")
    y = po.random_md(901 + m, m, 20000, "ref")
    assert_bitwise(po.random_md(900 + m, m, 20000, "port"), x, "random_md")
    for op in ("add", "sub", "mul"):
        assert_bitwise(po.md_op(op, x, y, "port"), po.md_op(op, x, y, "ref"), f"{op} m={m}")


@needs_ref
@pytest.mark.parametrize("pid", ["p1", "p2", "p3"])
def test_generator_and_graph_match_reference_library(pid):
    a = po.gen_benchmark(pid, 3, 2, seed=11)
    b = po.ref_gen_benchmark(pid, 3, 2, seed=11)
    assert_bitwise(a.stat, b.stat, "static")
    ga, gb = po.graph(a, "port"), po.graph(b, "ref")
    for k in ("conv", "add", "grad_slots", "mult"):
        assert (ga[k] == gb[k]).all(), k


@needs_ref
def test_random_instances_match_reference_library():
    rng = np.random.default_rng(77)
    for it in range(40):
        p = int_instance(rng, it % 2 == 0, cplx=it % 5 == 0)
        assert_bitwise(po.evaluate(p, "port"), po.evaluate(p, "ref"), f"int {it}")
        assert_bitwise(po.eval_direct(p, "port"), po.eval_direct(p, "ref"), f"direct {it}")
    for it, m in enumerate([2, 3, 4, 5, 8, 10] * 2):
        p = md_instance(rng, m, cplx=it % 2 == 1, with_exponents=it % 3 == 0)
        vg_p, dyn_p = po.evaluate(p, "port", want_dyn=True)
        vg_r, dyn_r = po.evaluate(p, "ref", want_dyn=True)
        assert_bitwise(vg_p, vg_r, f"md {it}")
        assert_bitwise(dyn_p, dyn_r, f"md arena {it}")


@needs_ref
def test_parallel_reference_equals_sequential():
    p = po.gen_benchmark("p1", 8, 2, seed=7)
    assert_bitwise(po.evaluate(p, "ref", workers=4), po.evaluate(p, "ref", workers=0))
