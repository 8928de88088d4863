"""Problem files (reference proj/src/problem_io.cpp, proj/tests/test_problem_io.cpp)
and the pseval_b200 CLI -- CPU only. The product's writer must produce the
reference's text byte for byte, and both parsers must accept each other's
files; parse errors carry the same line numbers and messages."""
import os
import subprocess

import numpy as np
import pytest

import paper_2101_10881_b200 as pe
from paper_2101_10881_b200 import pseval as ps
import pyoracle as po

needs_ref = pytest.mark.skipif(not po.has_ref(), reason="oracle/_ref not built")
CLI = os.path.join(os.path.dirname(pe.LIB_PATH), "pseval_b200")

SMALL = ("pseval 1\nproblem t 2 1 0 1 real 7\nconstant\n0x1p+0\nmonomial 2\nindices 1 2\n0x1p+1\n"
         "input 1\n0x1.8p+1\ninput 2\n0x1p+2\nend\n")


def with_line(text, lineno, repl):
    lines = text.split("\n")
    lines[lineno - 1] = repl
    return "\n".join(lines)


def same(a: ps.Problem, b: ps.Problem):
    assert (a.id, a.seed, a.n, a.d, a.m, a.mode) == (b.id, b.seed, b.n, b.d, b.m, b.mode)
    assert (a.nvars == b.nvars).all() and (a.indices == b.indices).all()
    assert (a.exponents is None) == (b.exponents is None)
    if a.exponents is not None:
        assert (a.exponents == b.exponents).all()
    assert (a.stat.view(np.uint64) == b.stat.view(np.uint64)).all()


def test_round_trip_reproduces_every_bit():
    p = pe.gen_benchmark("p1", 4, 2, "real", 12345)
    same(p, ps.problem_from_text(ps.problem_to_text(p)))


def test_round_trip_complex_with_exponents(tmp_path):
    rng = np.random.default_rng(3)
    stat = po.random_md(99, 5, 2 * 6 * 3).reshape(2, 6, 3, 5).transpose(0, 3, 1, 2).reshape(10, 6, 3).copy()
    p = ps.Problem("file", 99, 3, 2, 5, "cplx", np.array([2, 3], np.int32), np.array([1, 3, 1, 2, 3], np.int32),
                   stat, np.array([2, 1, 0, 0, 0], np.int32))
    q = ps.problem_from_text(ps.problem_to_text(p))
    same(p, q)
    path = str(tmp_path / "p.txt")
    ps.write_problem(path, p)
    same(p, ps.read_problem(path))
    assert "exponents 2 1" in open(path).read()


@needs_ref
@pytest.mark.parametrize("pid,d,m,cplx,seed", [("p1", 3, 2, False, 7), ("p2", 1, 3, True, 77), ("p3", 2, 10, False, 5)])
def test_writer_matches_reference_text_and_parsers_agree(pid, d, m, cplx, seed):
    ref_text = po.ref_problem_text(pid, d, m, cplx, seed)
    p = pe.gen_benchmark(pid, d, m, "cplx" if cplx else "real", seed)
    assert ps.problem_to_text(p) == ref_text
    same(p, ps.problem_from_text(ref_text))
    assert po.ref_parse_error(ps.problem_to_text(p)) == ""


def test_decimal_values_blank_lines_and_crlf():
    p = ps.problem_from_text(with_line(with_line(SMALL, 4, "1.5"), 9, "-0.25"))
    assert p.stat[0, 0, 0] == 1.5 and p.stat[0, 2, 0] == -0.25
    crlf = "".join(line + "\r\n\n" for line in SMALL.split("\n")[:-1])
    q = ps.problem_from_text(crlf)
    assert q.stat[0, 0, 0] == 1.0 and q.stat[0, 3, 0] == 4.0


CASES = [
    (1, "pseval 2", "not a pseval problem file", 1),
    (2, "problem t 2 1 0 7 real 7", "unsupported precision level", 2),
    (2, "problem t 2 1 0 1 quad 7", "unknown mode", 2),
    (6, "indices 1 1", "duplicate variable index", 6),
    (6, "indices 2 1", "indices must be strictly increasing", 6),
    (4, "0x1p+0 0x1p+0", "expected 1 values, got 2", 4),
    (4, "nope", "malformed number", 4),
    (12, "", "expected the end marker", None),
    (6, "indices 1 2\nexponents 0 1", "exponents must be positive", 7),
]


@pytest.mark.parametrize("lineno,repl,msg,line", CASES)
def test_parse_errors_carry_line_numbers(lineno, repl, msg, line):
    text = with_line(SMALL, lineno, repl)
    with pytest.raises(pe.InvalidArgument) as e:
        ps.problem_from_text(text)
    assert msg in str(e.value)
    if line is not None:
        assert f"line {line}:" in str(e.value)
    if po.has_ref():  # same message as the reference's ParseError
        assert po.ref_parse_error(text).split(": ", 1)[1] in str(e.value)


def test_unopenable_path_is_an_error():
    with pytest.raises(pe.PseError):
        ps.read_problem("no_such_directory/missing.txt")


# ---------------------------------------------------------------- CLI
def run_cli(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=120)


def test_cli_gen_and_graph_stats(tmp_path):
    out = str(tmp_path / "p1.txt")
    r = run_cli("gen", "p1", out, "--degree", "3", "--precision", "2")
    assert r.returncode == 0, r.stderr
    assert "wrote" in r.stdout
    same(ps.read_problem(out), pe.gen_benchmark("p1", 3, 2, "real", 7))
    r = run_cli("graph-stats", out)
    assert r.returncode == 0
    assert "conv jobs: 16380 in 4 layers: 3640 5460 5460 1820" in r.stdout
    assert "add jobs: 9084 in 11 layers: 4542 2279 1140 562 281 140 78 39 20 2 1" in r.stdout
    r = run_cli("graph-stats", "p3", "--degree", "2")
    assert "differs from the 24256" in r.stdout


def test_cli_errors():
    assert run_cli("frobnicate").returncode == 2
    assert run_cli("gen", "p9", "/tmp/x").returncode == 2
    r = run_cli("graph-stats", "no_such_file.txt")
    assert r.returncode == 2 and "cannot open" in r.stderr
