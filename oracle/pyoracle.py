"""TEST INFRASTRUCTURE ONLY -- the checker, never the product.

ctypes front end over the two CPU oracles:

* ``port``: the plain-C restatement ``oracle/pse_oracle.c`` (built into
  ``oracle/build/libpse_oracle.so``), and
* ``ref``: the reference engine itself, compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` into
  ``oracle/_ref/libpseval_ref.so`` (present wherever that library was built;
  it travels to the GPU box with the snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference leg import this module.

Array conventions (identical for both libraries and the product C ABI):
  static block  [P][m][1+N+n][d+1]   slot 0 = a0, 1+k = a_k, N+i = z_i
  value/grad    [P][m][n+1][d+1]     row 0 = value, 1+i = gradient of x_{i+1}
  md values     [count][m]
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "libpse_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpseval_ref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


@dataclass
class Problem:
    """A polynomial system + evaluation point in packed form (one point)."""

    n: int
    d: int
    m: int
    cplx: bool
    nvars: np.ndarray  # int32 [N]
    idx: np.ndarray  # int32 [sum nvars], 1-based
    exps: Optional[np.ndarray]  # int32 [sum nvars] or None
    stat: np.ndarray  # float64 [P][m][1+N+n][d+1]
    id: str = "file"

    @property
    def N(self) -> int:
        return int(self.nvars.shape[0])

    @property
    def P(self) -> int:
        return 2 if self.cplx else 1

    def monomials(self):
        out, pos = [], 0
        for k in range(self.N):
            nk = int(self.nvars[k])
            ix = [int(v) for v in self.idx[pos:pos + nk]]
            ex = None if self.exps is None else [int(v) for v in self.exps[pos:pos + nk]]
            if ex is not None and not any(ex):
                ex = None
            out.append((ix, ex))
            pos += nk
        return out


def has_ref() -> bool:
    return os.path.exists(REF_SO)


_port = None
_ref = None


def port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            raise RuntimeError(f"oracle port not built: {PORT_SO} (run make -C oracle)")
        L = C.CDLL(PORT_SO)
        L.pso_md_op.argtypes = [C.c_int, C.c_int, C.c_int64, _f64p, _f64p, _f64p]
        L.pso_cost.argtypes = [C.c_int, _i64p]
        L.pso_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.pso_mix_seed.restype = C.c_uint64
        L.pso_rng_u64.argtypes = [C.c_uint64, C.c_int64, _u64p]
        L.pso_random_md.argtypes = [C.c_uint64, C.c_int, C.c_int64, _f64p]
        L.pso_renormalize.argtypes = [_f64p, C.c_int, C.c_int, _f64p]
        L.pso_graph_build.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, _i32p, C.c_void_p]
        L.pso_graph_build.restype = C.c_void_p
        L.pso_graph_free.argtypes = [C.c_void_p]
        L.pso_graph_info.argtypes = [C.c_void_p, _i64p]
        L.pso_graph_export.argtypes = [C.c_void_p, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p]
        L.pso_graph_validate.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        L.pso_flop_count.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int]
        L.pso_flop_count.restype = C.c_int64
        L.pso_gen_shape_size.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.pso_gen_benchmark.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_uint64, _i32p, _i32p, C.c_void_p]
        L.pso_evaluate.argtypes = [C.c_int] * 5 + [_i32p, _i32p, C.c_void_p, _f64p, _f64p, C.c_void_p]
        L.pso_eval_direct.argtypes = [C.c_int] * 5 + [_i32p, _i32p, C.c_void_p, _f64p, _f64p]
        L.pso_series_conv.argtypes = [C.c_int, C.c_int, C.c_int, _f64p, _f64p, _f64p]
        L.pso_last_error.restype = C.c_char_p
        _port = L
    return _port


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference library not built: {REF_SO}")
        L = C.CDLL(REF_SO)
        L.ref_problem_gen.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_uint64]
        L.ref_problem_gen.restype = C.c_void_p
        L.ref_problem_new.argtypes = [C.c_int] * 5 + [_i32p, _i32p, C.c_void_p, _f64p]
        L.ref_problem_new.restype = C.c_void_p
        L.ref_problem_free.argtypes = [C.c_void_p]
        L.ref_problem_info.argtypes = [C.c_void_p, _i64p]
        L.ref_problem_shape.argtypes = [C.c_void_p, _i32p, _i32p, _i32p]
        L.ref_problem_static.argtypes = [C.c_void_p, _f64p]
        L.ref_graph_export.argtypes = [C.c_void_p, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p]
        L.ref_run.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_eval_direct.argtypes = [C.c_void_p, _f64p]
        L.ref_within_oracle_guard.argtypes = [C.c_void_p]
        L.ref_md_op.argtypes = [C.c_int, C.c_int, C.c_int64, _f64p, _f64p, _f64p]
        L.ref_random_md.argtypes = [C.c_uint64, C.c_int, C.c_int64, _f64p]
        L.ref_renormalize.argtypes = [_f64p, C.c_int, C.c_int, _f64p]
        L.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_mix_seed.restype = C.c_uint64
        L.ref_rng_u64.argtypes = [C.c_uint64, C.c_int64, _u64p]
        L.ref_cost.argtypes = [C.c_int, _i64p]
        L.ref_flop_count.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int]
        L.ref_flop_count.restype = C.c_int64
        L.ref_bench_sample.argtypes = [C.c_void_p, C.c_int, C.c_int64, _f64p]
        L.ref_run_bench.argtypes = [C.c_void_p, C.c_int, C.c_int, _f64p]
        L.ref_last_error.restype = C.c_char_p
        L.ref_problem_to_text.argtypes = [C.c_void_p, C.c_char_p, C.c_int64]
        L.ref_problem_to_text.restype = C.c_int64
        L.ref_problem_from_text.argtypes = [C.c_char_p]
        L.ref_problem_from_text.restype = C.c_void_p
        _ref = L
    return _ref


def _err(lib, which):
    msg = (lib.pso_last_error() if which == "port" else lib.ref_last_error()) or b""
    return RuntimeError(msg.decode())


# ----------------------------------------------------------------- md ops
def md_op(op: str, x: np.ndarray, y: np.ndarray, lib: str = "port") -> np.ndarray:
    """Elementwise exp_add/exp_sub/exp_mul over [count][m] arrays."""
    code = {"add": 0, "sub": 1, "mul": 2}[op]
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    count, m = x.shape
    out = np.empty_like(x)
    L = port_lib() if lib == "port" else ref_lib()
    f = L.pso_md_op if lib == "port" else L.ref_md_op
    if f(code, m, count, x, y, out) != 0:
        raise _err(L, lib)
    return out


def random_md(seed: int, m: int, count: int, lib: str = "port") -> np.ndarray:
    out = np.empty((count, m), np.float64)
    L = port_lib() if lib == "port" else ref_lib()
    (L.pso_random_md if lib == "port" else L.ref_random_md)(seed, m, count, out)
    return out


def renormalize(t, m: int, lib: str = "port") -> np.ndarray:
    t = np.ascontiguousarray(t, np.float64)
    out = np.zeros(m, np.float64)
    L = port_lib() if lib == "port" else ref_lib()
    f = L.pso_renormalize if lib == "port" else L.ref_renormalize
    if f(t, len(t), m, out) != 0:
        raise _err(L, lib)
    return out


def cost(m: int, lib: str = "port"):
    """(instrumented add, instrumented mul, reporting add, reporting mul)."""
    out = np.zeros(4, np.int64)
    L = port_lib() if lib == "port" else ref_lib()
    f = L.pso_cost if lib == "port" else L.ref_cost
    if f(m, out) != 0:
        raise _err(L, lib)
    return tuple(int(v) for v in out)


def mix_seed(base: int, stream: int, lib: str = "port") -> int:
    L = port_lib() if lib == "port" else ref_lib()
    return int((L.pso_mix_seed if lib == "port" else L.ref_mix_seed)(base, stream))


def rng_u64(seed: int, count: int, lib: str = "port") -> np.ndarray:
    out = np.empty(count, np.uint64)
    L = port_lib() if lib == "port" else ref_lib()
    (L.pso_rng_u64 if lib == "port" else L.ref_rng_u64)(seed, count, out)
    return out


def series_conv(x: np.ndarray, y: np.ndarray, cplx: bool = False) -> np.ndarray:
    """conv of two [P][m][d+1] series (port only)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    out = np.empty_like(x)
    P, m, d1 = x.shape
    if port_lib().pso_series_conv(d1 - 1, m, int(cplx), x, y, out) != 0:
        raise _err(port_lib(), "port")
    return out


# ----------------------------------------------------------------- problems
def gen_benchmark(pid: str, d: int, m: int, cplx: bool = False, seed: int = 7, with_static: bool = True) -> Problem:
    """gen_benchmark (gen.cpp:50-71) via the C restatement."""
    L = port_lib()
    n, N, ln = C.c_int(), C.c_int(), C.c_int()
    if L.pso_gen_shape_size(pid.encode(), C.byref(n), C.byref(N), C.byref(ln)) != 0:
        raise _err(L, "port")
    nvars = np.empty(N.value, np.int32)
    idx = np.empty(ln.value, np.int32)
    P = 2 if cplx else 1
    stat = np.empty((P, m, 1 + N.value + n.value, d + 1), np.float64) if with_static else None
    rc = L.pso_gen_benchmark(pid.encode(), d, m, int(cplx), seed, nvars, idx,
                             stat.ctypes.data if stat is not None else None)
    if rc != 0:
        raise _err(L, "port")
    return Problem(n.value, d, m, cplx, nvars, idx, None, stat, pid)


def ref_gen_benchmark(pid: str, d: int, m: int, cplx: bool = False, seed: int = 7) -> Problem:
    """gen_benchmark run by the reference library itself."""
    L = ref_lib()
    h = L.ref_problem_gen(pid.encode(), d, m, int(cplx), seed)
    if not h:
        raise _err(L, "ref")
    try:
        info = np.zeros(13, np.int64)
        L.ref_problem_info(h, info)
        n, N = int(info[0]), int(info[1])
        nvars = np.empty(N, np.int32)
        idx = np.empty(int(info[12]), np.int32)
        exps = np.empty(int(info[12]), np.int32)
        L.ref_problem_shape(h, nvars, idx, exps)
        P = 2 if cplx else 1
        stat = np.empty((P, m, 1 + N + n, d + 1), np.float64)
        L.ref_problem_static(h, stat)
        return Problem(n, d, m, cplx, nvars, idx, exps if exps.any() else None, stat, pid)
    finally:
        L.ref_problem_free(h)


def _exps_ptr(p: Problem):
    if p.exps is None:
        return None, None
    e = np.ascontiguousarray(p.exps, np.int32)
    return e, e.ctypes.data


def _ref_handle(p: Problem):
    L = ref_lib()
    e, ep = _exps_ptr(p)
    stat = np.ascontiguousarray(p.stat, np.float64)
    h = L.ref_problem_new(p.n, p.d, p.m, int(p.cplx), p.N, np.ascontiguousarray(p.nvars, np.int32),
                          np.ascontiguousarray(p.idx, np.int32), ep, stat)
    if not h:
        raise _err(L, "ref")
    return h


def vg_shape(p: Problem):
    return (p.P, p.m, p.n + 1, p.d + 1)


def evaluate(p: Problem, lib: str = "port", workers: int = 0, want_dyn: bool = False):
    """evaluate() (executor.cpp:271-276). Returns vg [P][m][n+1][d+1] (and the
    full arena [P][m][total_slots][d+1] when want_dyn)."""
    vg = np.empty(vg_shape(p), np.float64)
    if lib == "port":
        L = port_lib()
        dyn = None
        if want_dyn:
            g = graph(p, "port")
            dyn = np.empty((p.P, p.m, g["total_slots"], p.d + 1), np.float64)
        e, ep = _exps_ptr(p)
        rc = L.pso_evaluate(p.n, p.d, p.m, int(p.cplx), p.N, np.ascontiguousarray(p.nvars, np.int32),
                            np.ascontiguousarray(p.idx, np.int32), ep, np.ascontiguousarray(p.stat), vg,
                            dyn.ctypes.data if dyn is not None else None)
        if rc != 0:
            raise _err(L, "port")
        return (vg, dyn) if want_dyn else vg
    L = ref_lib()
    h = _ref_handle(p)
    try:
        dyn = None
        if want_dyn:
            info = np.zeros(13, np.int64)
            L.ref_problem_info(h, info)
            dyn = np.empty((p.P, p.m, int(info[5]), p.d + 1), np.float64)
        times = np.zeros(3, np.float64)
        ops = np.zeros(1, np.int64)
        if L.ref_run(h, workers, vg.ctypes.data, dyn.ctypes.data if dyn is not None else None,
                     times.ctypes.data, ops.ctypes.data) != 0:
            raise _err(L, "ref")
        return (vg, dyn) if want_dyn else vg
    finally:
        L.ref_problem_free(h)


def eval_direct(p: Problem, lib: str = "port"):
    vg = np.empty(vg_shape(p), np.float64)
    if lib == "port":
        L = port_lib()
        e, ep = _exps_ptr(p)
        rc = L.pso_eval_direct(p.n, p.d, p.m, int(p.cplx), p.N, np.ascontiguousarray(p.nvars, np.int32),
                               np.ascontiguousarray(p.idx, np.int32), ep, np.ascontiguousarray(p.stat), vg)
        if rc != 0:
            raise _err(L, "port")
        return vg
    L = ref_lib()
    h = _ref_handle(p)
    try:
        if L.ref_eval_direct(h, vg) != 0:
            raise _err(L, "ref")
        return vg
    finally:
        L.ref_problem_free(h)


def graph(p: Problem, lib: str = "port") -> dict:
    """Flattened JobGraph: conv rows (layer,in1,in2,out,copy), add rows
    (layer,src,dst), value slot, gradient slots, multipliers, term scales."""
    e, ep = _exps_ptr(p)
    if lib == "port":
        L = port_lib()
        g = L.pso_graph_build(p.n, p.d, p.N, np.ascontiguousarray(p.nvars, np.int32),
                              np.ascontiguousarray(p.idx, np.int32), ep)
        if not g:
            raise _err(L, "port")
        try:
            info = np.zeros(10, np.int64)
            L.pso_graph_info(g, info)
            n, N, d, ts_, nconv, nadd, ncopy, ncl, nal, nts = (int(v) for v in info)
            conv = np.empty((nconv, 5), np.int64)
            add = np.empty((nadd, 3), np.int64)
            vs = np.zeros(1, np.int64)
            gs = np.empty(n, np.int64)
            mu = np.empty(n, np.int64)
            tsa = np.empty((max(nts, 1), 2), np.int64)
            L.pso_graph_export(g, conv, add, vs, gs, mu, tsa)
            msg = C.create_string_buffer(512)
            ok = L.pso_graph_validate(g, msg, 512)
            flops = {}
            return dict(total_slots=ts_, conv=conv, add=add, value_slot=int(vs[0]), grad_slots=gs, mult=mu,
                        term_scales=tsa[:nts], n_conv_layers=ncl, n_add_layers=nal, ncopy=ncopy,
                        valid=bool(ok), message=msg.value.decode(), _flops=flops)
        finally:
            L.pso_graph_free(g)
    L = ref_lib()
    h = _ref_handle(p)
    try:
        info = np.zeros(13, np.int64)
        L.ref_problem_info(h, info)
        n = int(info[0])
        conv = np.empty((int(info[6]), 5), np.int64)
        add = np.empty((int(info[7]), 3), np.int64)
        nts = int(info[11])
        vs = np.zeros(1, np.int64)
        gs = np.empty(n, np.int64)
        mu = np.empty(n, np.int64)
        tsa = np.empty((max(nts, 1), 2), np.int64)
        L.ref_graph_export(h, conv, add, vs, gs, mu, tsa)
        return dict(total_slots=int(info[5]), conv=conv, add=add, value_slot=int(vs[0]), grad_slots=gs, mult=mu,
                    term_scales=tsa[:nts], n_conv_layers=int(info[9]), n_add_layers=int(info[10]),
                    ncopy=int(info[8]))
    finally:
        L.ref_problem_free(h)


def flop_count(p: Problem, add_cost: int, mul_cost: int, which: int = 0, lib: str = "port", d: Optional[int] = None) -> int:
    d = p.d if d is None else d
    e, ep = _exps_ptr(p)
    if lib == "port":
        L = port_lib()
        g = L.pso_graph_build(p.n, p.d, p.N, np.ascontiguousarray(p.nvars, np.int32),
                              np.ascontiguousarray(p.idx, np.int32), ep)
        try:
            return int(L.pso_flop_count(g, d, int(p.cplx), add_cost, mul_cost, which))
        finally:
            L.pso_graph_free(g)
    L = ref_lib()
    h = _ref_handle(p)
    try:
        return int(L.ref_flop_count(h, d, int(p.cplx), add_cost, mul_cost, which))
    finally:
        L.ref_problem_free(h)


def ref_problem_text(pid: str, d: int, m: int, cplx: bool = False, seed: int = 7) -> str:
    """problem_to_text(gen_benchmark(...)) by the reference library."""
    L = ref_lib()
    h = L.ref_problem_gen(pid.encode(), d, m, int(cplx), seed)
    if not h:
        raise _err(L, "ref")
    try:
        n = L.ref_problem_to_text(h, None, 0)
        buf = C.create_string_buffer(n + 1)
        L.ref_problem_to_text(h, buf, n + 1)
        return buf.value.decode()
    finally:
        L.ref_problem_free(h)


def ref_problem_text_of(p: Problem) -> str:
    """problem_to_text of an arbitrary packed problem (id 'file', seed 0)."""
    L = ref_lib()
    h = _ref_handle(p)
    try:
        n = L.ref_problem_to_text(h, None, 0)
        buf = C.create_string_buffer(n + 1)
        L.ref_problem_to_text(h, buf, n + 1)
        return buf.value.decode()
    finally:
        L.ref_problem_free(h)


def ref_parse_error(text: str) -> str:
    """'' if the reference parses text, else its ParseError message."""
    L = ref_lib()
    h = L.ref_problem_from_text(text.encode())
    if h:
        L.ref_problem_free(h)
        return ""
    return (L.ref_last_error() or b"").decode()


# ----------------------------------------------------------------- CPU timing
def ref_run_bench(p: Problem, workers: int, repeats: int = 3):
    """The reference's own run_bench (bench.cpp:17-50) on the whole graph:
    returns (conv_ms, add_ms, wall_ms, gflops)."""
    L = ref_lib()
    h = _ref_handle(p)
    try:
        out = np.zeros(4, np.float64)
        if L.ref_run_bench(h, workers, repeats, out) != 0:
            raise _err(L, "ref")
        return tuple(float(v) for v in out)
    finally:
        L.ref_problem_free(h)


def ref_bench_sample(p: Problem, workers: int, njobs: int):
    """Reference run_parallel over the first njobs conv jobs of layer 1 plus all
    add layers; returns (conv_ms, add_ms, wall_ms, jobs_run)."""
    L = ref_lib()
    h = _ref_handle(p)
    try:
        t = np.zeros(3, np.float64)
        jobs = L.ref_bench_sample(h, workers, njobs, t)
        if jobs < 0:
            raise _err(L, "ref")
        return float(t[0]), float(t[1]), float(t[2]), int(jobs)
    finally:
        L.ref_problem_free(h)


def port_time_conv_jobs(p: Problem, njobs: int) -> tuple[float, int]:
    """Fallback CPU timer when the reference library is absent: the C port's
    series conv on the first njobs layer-1 conv jobs, single thread.
    Returns (ms, jobs_run)."""
    import time

    g = graph(p, "port")
    rows = [r for r in g["conv"] if r[0] == 1 and r[4] == 0][:njobs]
    top = 1 + p.N + p.n
    t0 = time.perf_counter()
    for r in rows:
        a, b = int(r[1]), int(r[2])
        if a >= top or b >= top:
            continue
        series_conv(p.stat[:, :, a, :], p.stat[:, :, b, :], p.cplx)
    return (time.perf_counter() - t0) * 1e3, len(rows)
