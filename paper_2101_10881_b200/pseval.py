"""Python mirror of the reference ``pseval`` API over the native C ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/pseval/*.hpp); the work happens in
``libpse_b200.so`` (graph compiler in C++, engine in CUDA for sm_100a).

Series are numpy arrays of shape [P][m][d+1] (P = 2 parts re/im in complex
mode, else 1): limb-split structure-of-arrays, limb 0 most significant.

    reference                               here
    ---------------------------------------------------------------------
    Polynomial / Monomial (jobgraph.hpp:26-37)   Polynomial / Monomial
    build_jobgraph (jobgraph.cpp:199-262)        build_jobgraph -> JobGraph
    validate (jobgraph.cpp:273-336)              validate
    stage (executor.cpp:69-96)                   stage -> DataArray
    run_sequential / run_parallel                run_device(graph, data)
      (executor.cpp:168-231)
    extract (executor.cpp:254-269)               part of run_device / evaluate
    evaluate (executor.cpp:271-276)              evaluate(poly, z)
    flop_count* (executor.cpp:233-252)           flop_count, flop_count_mul, flop_count_add
    instrumented_cost / reporting_cost           instrumented_cost / reporting_cost
    gen_benchmark (gen.cpp:50-71)                gen_benchmark -> Problem
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import GraphDesc, InvalidArgument, Report, check, lib, ptr, ptr_array

REAL = "real"
CPLX = "cplx"
PRECISION_LEVELS = (1, 2, 3, 4, 5, 8, 10)  # kPrecisionLevels, multidouble.hpp:20


def _mode_code(mode: str) -> int:
    if mode in (REAL, "real", 0):
        return _lib.PSE_MODE_REAL
    if mode in (CPLX, "cplx", "complex", 1):
        return _lib.PSE_MODE_COMPLEX
    raise InvalidArgument(-1, f"unknown mode {mode!r}")


def check_precision(m: int) -> None:
    if m not in PRECISION_LEVELS:
        raise InvalidArgument(-1, "unsupported precision level")


# ----------------------------------------------------------------- series
def make_series(degree: int, m: int, mode: str = REAL) -> np.ndarray:
    if degree < 0:
        raise InvalidArgument(-1, "negative truncation degree")
    check_precision(m)
    return np.zeros((2 if _mode_code(mode) else 1, m, degree + 1), np.float64)


def one_series(degree: int, m: int, mode: str = REAL) -> np.ndarray:
    s = make_series(degree, m, mode)
    s[0, 0, 0] = 1.0
    return s


def series_bitwise_equal(x: np.ndarray, y: np.ndarray) -> bool:
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    return x.shape == y.shape and bool((x.view(np.uint64) == y.view(np.uint64)).all())


# ----------------------------------------------------------------- polynomials
@dataclass
class Monomial:
    coeff: np.ndarray  # [P][m][d+1]
    indices: List[int]  # strictly increasing, 1-based
    exponents: Optional[List[int]] = None  # None/empty = all 1


@dataclass
class Polynomial:
    n: int
    d: int
    a0: np.ndarray  # [P][m][d+1]
    monomials: List[Monomial] = field(default_factory=list)

    @property
    def m(self) -> int:
        return int(self.a0.shape[1])

    @property
    def mode(self) -> str:
        return CPLX if self.a0.shape[0] == 2 else REAL

    def shape_arrays(self):
        nv = np.array([len(mo.indices) for mo in self.monomials], np.int32)
        idx = np.array([i for mo in self.monomials for i in mo.indices], np.int32)
        has = any(mo.exponents for mo in self.monomials)
        ex = None
        if has:
            ex = np.array([e for mo in self.monomials
                           for e in (mo.exponents if mo.exponents else [0] * len(mo.indices))], np.int32)
        return nv, idx, ex


def check_polynomial(p: Polynomial) -> None:
    """check_polynomial (jobgraph.cpp:41-63), plus the series agreement checks."""
    if p.n < 1:
        raise InvalidArgument(-1, "polynomial needs at least one variable")
    if not p.monomials:
        raise InvalidArgument(-1, "polynomial needs at least one monomial")
    if p.a0.shape[2] != p.d + 1:
        raise InvalidArgument(-1, "constant term degree mismatch")
    for mo in p.monomials:
        if not mo.indices:
            raise InvalidArgument(-1, "monomial without variables")
        if mo.coeff.shape != p.a0.shape:
            raise InvalidArgument(-1, "monomial coefficient series mismatch")
        if mo.exponents and len(mo.exponents) != len(mo.indices):
            raise InvalidArgument(-1, "exponent count mismatch")


# ----------------------------------------------------------------- job graph
class JobGraph:
    """Compiled job graph (jobgraph.hpp:75-90) owned by the native library."""

    def __init__(self, handle: int, n: int, N: int, d: int):
        self._h = C.c_void_p(handle)
        self.n, self.N, self.d = n, N, d
        desc = self.desc(1, REAL)
        self.total_slots = int(desc.total_slots)
        self.value_slot = int(desc.value_slot)
        nl, al = int(desc.n_conv_layers), int(desc.n_add_layers)
        coff = np.ctypeslib.as_array(desc.conv_layer_off, (nl + 1,)).copy()
        aoff = np.ctypeslib.as_array(desc.add_layer_off, (al + 1,)).copy()
        nc, na = int(coff[-1]), int(aoff[-1])
        arr = lambda p, k: np.ctypeslib.as_array(p, (k,)).copy() if k else np.zeros(0, np.int64)
        self.conv_layer_off, self.add_layer_off = coff, aoff
        self.conv_in1, self.conv_in2, self.conv_out = arr(desc.conv_in1, nc), arr(desc.conv_in2, nc), arr(desc.conv_out, nc)
        self.conv_copy = arr(desc.conv_copy, nc).astype(bool)
        self.add_src, self.add_dst = arr(desc.add_src, na), arr(desc.add_dst, na)
        self.gradient_slots = arr(desc.gradient_slots, n)
        self.multipliers = arr(desc.multipliers, n)
        nts = int(desc.n_term_scales)
        self.term_scales = np.stack([arr(desc.ts_slot, nts), arr(desc.ts_factor, nts)], 1) if nts else np.zeros((0, 2), np.int64)

    def desc(self, m: int, mode: str) -> GraphDesc:
        d = GraphDesc()
        check(lib().pse_graph_describe(self._h, m, _mode_code(mode), C.byref(d)))
        return d

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().pse_graph_destroy(h)
            self._h = C.c_void_p(0)

    # reference accessors (jobgraph.cpp:9-37)
    def conv_job_count(self) -> int:
        return int(self.conv_layer_off[-1])

    def add_job_count(self) -> int:
        return int(self.add_layer_off[-1])

    def copy_job_count(self) -> int:
        return int(self.conv_copy.sum())

    def conv_layer_sizes(self) -> List[int]:
        return [int(v) for v in np.diff(self.conv_layer_off)]

    def add_layer_sizes(self) -> List[int]:
        return [int(v) for v in np.diff(self.add_layer_off)]

    @property
    def conv_layers(self):
        """list of layers of (in1, in2, out, layer, copy) tuples."""
        out = []
        for L in range(len(self.conv_layer_off) - 1):
            a, b = self.conv_layer_off[L], self.conv_layer_off[L + 1]
            out.append([(int(self.conv_in1[t]), int(self.conv_in2[t]), int(self.conv_out[t]), L + 1,
                         bool(self.conv_copy[t])) for t in range(a, b)])
        return out

    @property
    def add_layers(self):
        """list of layers of (src, dst, layer) tuples."""
        out = []
        for L in range(len(self.add_layer_off) - 1):
            a, b = self.add_layer_off[L], self.add_layer_off[L + 1]
            out.append([(int(self.add_src[t]), int(self.add_dst[t]), L + 1) for t in range(a, b)])
        return out


class GraphArrays:
    """A pse_graph_desc over caller-owned numpy arrays (e.g. a JobGraph read
    back, edited, and handed to validate() or a DevicePlan)."""

    def __init__(self, n, N, d, total_slots, value_slot, gradient_slots, multipliers, conv_layer_off, conv_in1,
                 conv_in2, conv_out, conv_copy, add_layer_off, add_src, add_dst, ts_slot=(), ts_factor=()):
        i64 = lambda a: np.ascontiguousarray(a, np.int64)
        self._keep = dict(gs=i64(gradient_slots), mu=i64(multipliers), co=i64(conv_layer_off), c1=i64(conv_in1),
                          c2=i64(conv_in2), c3=i64(conv_out), cc=np.ascontiguousarray(conv_copy, np.uint8),
                          ao=i64(add_layer_off), a1=i64(add_src), a2=i64(add_dst), t1=i64(ts_slot), t2=i64(ts_factor))
        k = self._keep
        P64, P8 = C.POINTER(C.c_int64), C.POINTER(C.c_uint8)
        p = lambda a, t=P64: a.ctypes.data_as(t)
        self.n, self.N, self.d, self.total_slots = n, N, d, total_slots
        self.desc_base = dict(n=n, N=N, d=d, total_slots=total_slots, value_slot=value_slot, gradient_slots=p(k["gs"]),
                              multipliers=p(k["mu"]), n_conv_layers=len(k["co"]) - 1, conv_layer_off=p(k["co"]),
                              conv_in1=p(k["c1"]), conv_in2=p(k["c2"]), conv_out=p(k["c3"]), conv_copy=p(k["cc"], P8),
                              n_add_layers=len(k["ao"]) - 1, add_layer_off=p(k["ao"]), add_src=p(k["a1"]),
                              add_dst=p(k["a2"]), n_term_scales=len(k["t1"]), ts_slot=p(k["t1"]), ts_factor=p(k["t2"]))

    @classmethod
    def from_graph(cls, g: "JobGraph"):
        return cls(g.n, g.N, g.d, g.total_slots, g.value_slot, g.gradient_slots, g.multipliers, g.conv_layer_off,
                   g.conv_in1, g.conv_in2, g.conv_out, g.conv_copy, g.add_layer_off, g.add_src, g.add_dst,
                   g.term_scales[:, 0], g.term_scales[:, 1])

    def desc(self, m: int, mode: str) -> GraphDesc:
        d = GraphDesc(**self.desc_base)
        d.m, d.mode = m, _mode_code(mode)
        return d


def band_schedule_stats(g, W: int, flow: bool = True, procs: int = 2368, slack: float = 0.3) -> dict:
    """The banded conv schedule of graph g (host only, pse_band_schedule_stats):
    task and descriptor counts of the dataflow order (flow) or of waves of
    `procs` warps; raises if a descriptor would wait on a later one."""
    out = np.zeros(7, np.int64)
    d = g.desc(1, REAL)
    check(lib().pse_band_schedule_stats(C.byref(d), W, int(flow), procs, slack, out.ctypes.data))
    keys = ("jobs", "tasks", "descriptors", "waves", "dep_entries", "slots", "makespan_steps")
    return dict(zip(keys, (int(v) for v in out)))


def build_jobgraph_shape(n: int, d: int, nvars, indices, exponents=None) -> JobGraph:
    nv = np.ascontiguousarray(nvars, np.int32)
    ix = np.ascontiguousarray(indices, np.int32)
    ex = None if exponents is None else np.ascontiguousarray(exponents, np.int32)
    h = C.c_void_p()
    check(lib().pse_graph_build(n, d, len(nv), ptr(nv), ptr(ix), ptr(ex), C.byref(h)))
    return JobGraph(h.value, n, len(nv), d)


def build_jobgraph(p: Polynomial) -> JobGraph:
    check_polynomial(p)
    nv, idx, ex = p.shape_arrays()
    return build_jobgraph_shape(p.n, p.d, nv, idx, ex)


def validate(g: JobGraph, m: int = 1, mode: str = REAL):
    """(ok, message) -- validate (jobgraph.cpp:273-336)."""
    d = g.desc(m, mode)
    msg = C.create_string_buffer(512)
    rc = check(lib().pse_graph_validate(C.byref(d), msg, 512))
    return rc == 1, msg.value.decode()


# ----------------------------------------------------------------- costs
@dataclass
class OpCost:
    add_cost: int
    mul_cost: int


def _costs(m: int):
    out = np.zeros(4, np.int64)
    check(lib().pse_cost(m, ptr(out)))
    return out


def instrumented_cost(m: int) -> OpCost:
    c = _costs(m)
    return OpCost(int(c[0]), int(c[1]))


def reporting_cost(m: int) -> OpCost:
    c = _costs(m)
    return OpCost(int(c[2]), int(c[3]))


def flop_count(g: JobGraph, d: int, mode: str, cost: OpCost, which: int = 0) -> int:
    desc = g.desc(1, mode)
    desc.d = d
    return int(lib().pse_flop_count(C.byref(desc), which, cost.add_cost, cost.mul_cost))


def flop_count_mul(g: JobGraph, d: int, mode: str, cost: OpCost) -> int:
    return flop_count(g, d, mode, cost, 1)


def flop_count_add(g: JobGraph, d: int, mode: str, cost: OpCost) -> int:
    return flop_count(g, d, mode, cost, 2)


# ----------------------------------------------------------------- data
@dataclass
class DataArray:
    """Reference DataArray (executor.hpp:17-29): slab q (= part*m + limb)
    holds slot s coefficient j at [q][s][j]."""

    d: int
    m: int
    mode: str
    total_slots: int
    slabs: np.ndarray  # [Q][total_slots][d+1]

    def stride(self) -> int:
        return self.d + 1

    def read_slot(self, slot: int) -> np.ndarray:
        P = 2 if self.mode == CPLX else 1
        return self.slabs[:, slot, :].reshape(P, self.m, self.d + 1).copy()


def static_block(p: Polynomial, z: Sequence[np.ndarray]) -> np.ndarray:
    """Packed static region [Q][1+N+n][d+1] (slot 0 a0, 1+k a_k, N+i z_i)."""
    Q = p.a0.shape[0] * p.m
    N = len(p.monomials)
    out = np.empty((Q, 1 + N + p.n, p.d + 1), np.float64)
    out[:, 0] = p.a0.reshape(Q, -1)
    for k, mo in enumerate(p.monomials):
        out[:, 1 + k] = mo.coeff.reshape(Q, -1)
    for i, zi in enumerate(z):
        out[:, 1 + N + i] = np.asarray(zi).reshape(Q, -1)
    return out


def _check_inputs(p: Polynomial, z: Sequence[np.ndarray]):
    check_polynomial(p)
    if len(z) != p.n:
        raise InvalidArgument(-1, "input series count does not match the variable count")
    for zi in z:
        zi = np.asarray(zi)
        if zi.shape[2] != p.d + 1:
            raise InvalidArgument(-1, "input series degree mismatch")
        if zi.shape[1] != p.m:
            raise InvalidArgument(-1, "input series precision mismatch")
        if zi.shape[0] != p.a0.shape[0]:
            raise InvalidArgument(-1, "input series mode mismatch")


def stage(p: Polynomial, z: Sequence[np.ndarray]) -> DataArray:
    """stage (executor.cpp:69-96): static region filled, dynamic zeroed."""
    _check_inputs(p, z)
    for mo in p.monomials:
        if mo.exponents and any(e != 1 for e in mo.exponents):
            raise InvalidArgument(-1, "stage expects exponent-folded coefficients")
    g = build_jobgraph(p)
    Q = p.a0.shape[0] * p.m
    slabs = np.zeros((Q, g.total_slots, p.d + 1), np.float64)
    st = static_block(p, z)
    slabs[:, : st.shape[1]] = st
    return DataArray(p.d, p.m, p.mode, g.total_slots, slabs)


@dataclass
class RunReport:
    value: np.ndarray  # [P][m][d+1]
    gradient: List[np.ndarray]
    wall_ms: float = 0.0
    conv_ms: float = 0.0
    add_ms: float = 0.0
    scale_ms: float = 0.0
    h2d_ms: float = 0.0
    d2h_ms: float = 0.0
    e2e_ms: float = 0.0
    double_op_count: int = 0
    alg_op_count: int = 0
    conv_jobs_executed: int = 0
    add_jobs_executed: int = 0
    kernel_launches: int = 0
    conv_layer_ms: List[float] = field(default_factory=list)  # executor.hpp:31-43
    add_layer_ms: List[float] = field(default_factory=list)
    device_ms: float = 0.0


def _split_vg(vg: np.ndarray, P: int, m: int, n: int, d: int):
    """vg [Q][n+1][d+1] -> (value, [gradients]) as [P][m][d+1] series."""
    v = vg.reshape(P, m, n + 1, d + 1)
    return v[:, :, 0, :].copy(), [v[:, :, 1 + i, :].copy() for i in range(n)]


# ----------------------------------------------------------------- device plan
class DevicePlan:
    """A job graph resident on one GPU with an arena for up to max_batch
    points (pse_plan_*)."""

    def __init__(self, g: JobGraph, m: int, mode: str = REAL, device: int = 0, max_batch: int = 1,
                 rank: int = 0, nranks: int = 1):
        """rank/nranks > 1: this plan is rank's share of one polynomial sharded
        over nranks devices (pse_plan_create_sharded)."""
        check_precision(m)
        self.graph, self.m, self.mode, self.device, self.max_batch = g, m, mode, device, max_batch
        self.rank, self.nranks = rank, nranks
        self.P = 2 if _mode_code(mode) else 1
        self.Q = self.P * m
        self.top = 1 + g.N + g.n
        self._desc = g.desc(m, mode)
        h = C.c_void_p()
        if nranks > 1:
            check(lib().pse_plan_create_sharded(C.byref(self._desc), device, max_batch, rank, nranks, C.byref(h)))
        else:
            check(lib().pse_plan_create(C.byref(self._desc), device, max_batch, C.byref(h)))
        self._h = h

    # ---- sharded evaluation (see include/pse_b200.h)
    def exchange_words(self, rank: int, batch: int = 1) -> int:
        w = C.c_int64()
        check(lib().pse_plan_exchange_words(self._h, rank, batch, C.byref(w)))
        return w.value

    def pack(self, dst_ptr: int, batch: int = 1):
        check(lib().pse_plan_pack(self._h, batch, dst_ptr))

    def unpack(self, src_rank: int, src_ptr: int, batch: int = 1):
        check(lib().pse_plan_unpack(self._h, batch, src_rank, src_ptr))

    def ipc_handle(self) -> bytes:
        """CUDA IPC handle of this plan's arena (pse_plan_arena_ipc_handle)"""
        buf = C.create_string_buffer(64)
        check(lib().pse_plan_arena_ipc_handle(self._h, buf))
        return buf.raw

    def open_peer(self, rank: int, handle: bytes):
        """map rank's arena from its IPC handle (another process)"""
        buf = C.create_string_buffer(bytes(handle), 64)
        check(lib().pse_plan_open_peer(self._h, rank, buf))

    def set_peer(self, rank: int, peer: "DevicePlan"):
        """use another plan of this process as rank's arena"""
        check(lib().pse_plan_set_peer_arena(self._h, rank, peer._h))

    def gather_peers(self, batch: int = 1):
        """copy the slots the peers produced from their arenas (after a barrier)"""
        check(lib().pse_plan_gather_peers(self._h, batch))

    def finish(self, batch: int = 1, detail: bool = True) -> Report:
        rep = Report()
        check(lib().pse_plan_finish(self._h, batch, int(detail), C.byref(rep)))
        return rep

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().pse_plan_destroy(self._h)
            self._h = C.c_void_p(0)

    def __del__(self):
        self.close()

    def _slabs(self, stat: np.ndarray, batch: int):
        """stat: [Q][batch][top][d+1] contiguous (or [Q][top][d+1] when batch 1)."""
        stat = np.ascontiguousarray(stat, np.float64)
        pw = self.top * (self.graph.d + 1)
        base = stat.ctypes.data
        return stat, ptr_array([base + q * batch * pw * 8 for q in range(self.Q)])

    def upload(self, stat: np.ndarray, batch: int = 1):
        stat, slabs = self._slabs(stat, batch)
        check(lib().pse_plan_upload(self._h, batch, slabs, 0))

    def upload_ptr(self, base: int, batch: int, total: int = None, first: int = 0):
        """Stage points [first, first+batch) of a contiguous [Q][total][top][d+1]
        buffer at address `base` -- host or device memory (e.g. a CUDA tensor's
        data_ptr(): inputs resident in HBM are staged with a D2D copy)."""
        total = batch if total is None else total
        pw = self.top * (self.graph.d + 1)
        slabs = ptr_array([base + (q * total + first) * pw * 8 for q in range(self.Q)])
        check(lib().pse_plan_upload(self._h, batch, slabs, 0))

    def stream(self) -> int:
        """the plan's cudaStream_t as an integer handle"""
        s = C.c_void_p()
        check(lib().pse_plan_stream(self._h, C.byref(s)))
        return s.value or 0

    CONV_PATHS = {1: "layered", 2: "waves", 3: "dataflow", 4: "hybrid", 5: "cta", 6: "cta_layers"}

    def conv_path(self, batch: int = 1) -> str:
        """the convolution path a run of `batch` points takes
        (pse_plan_conv_path): layered, waves, dataflow or hybrid"""
        v = C.c_int32()
        check(lib().pse_plan_conv_path(self._h, batch, C.byref(v)))
        return self.CONV_PATHS[v.value]

    def execute(self, batch: int = 1, detail: bool = False) -> Report:
        rep = Report()
        check(lib().pse_plan_execute(self._h, batch, int(detail), C.byref(rep)))
        return rep

    def layer_ms(self):
        """(conv_layer_ms, add_layer_ms) of the last run (pse_plan_layer_ms;
        RunReport's per-phase lists, executor.cpp:154-157)"""
        nc, na = int(self._desc.n_conv_layers), int(self._desc.n_add_layers)
        c, a = np.zeros(nc), np.zeros(na)
        check(lib().pse_plan_layer_ms(self._h, ptr(c), nc, ptr(a), na))
        return [float(x) for x in c], [float(x) for x in a]

    def download(self, batch: int = 1, want_dyn: bool = False, out: Optional[np.ndarray] = None):
        """(vg [Q][batch][n+1][d+1], dyn or None); out: a caller-owned
        (e.g. pinned) C-contiguous array of vg's shape to write into"""
        n, d = self.graph.n, self.graph.d
        vg = out if out is not None else np.empty((self.Q, batch, n + 1, d + 1), np.float64)
        vw = batch * (n + 1) * (d + 1)
        vptr = ptr_array([vg.ctypes.data + q * vw * 8 for q in range(self.Q)])
        dyn, dptr = None, None
        if want_dyn:
            TS = self.graph.total_slots
            dyn = np.empty((self.Q, batch, TS, d + 1), np.float64)
            dw = batch * TS * (d + 1)
            dptr = ptr_array([dyn.ctypes.data + q * dw * 8 for q in range(self.Q)])
        check(lib().pse_plan_download(self._h, batch, vptr, dptr))
        return vg, dyn

    def run(self, stat: np.ndarray, batch: int = 1, out: Optional[np.ndarray] = None, want_dyn: bool = False):
        """upload + execute + download in one C-ABI call. Returns (vg, dyn, Report)."""
        n, d = self.graph.n, self.graph.d
        stat, slabs = self._slabs(stat, batch)
        vg = out if out is not None else np.empty((self.Q, batch, n + 1, d + 1), np.float64)
        vw = batch * (n + 1) * (d + 1)
        vptr = ptr_array([vg.ctypes.data + q * vw * 8 for q in range(self.Q)])
        dyn, dptr = None, None
        if want_dyn:
            TS = self.graph.total_slots
            dyn = np.empty((self.Q, batch, TS, d + 1), np.float64)
            dw = batch * TS * (d + 1)
            dptr = ptr_array([dyn.ctypes.data + q * dw * 8 for q in range(self.Q)])
        rep = Report()
        check(lib().pse_plan_run(self._h, batch, slabs, 0, dptr, vptr, C.byref(rep)))
        return vg, dyn, rep


def run_device(g: JobGraph, a: DataArray, device: int = 0) -> RunReport:
    """run_sequential's contract (executor.hpp:49) on the GPU: reads the
    static region of `a`, writes the whole dynamic region back into `a`,
    returns value and gradient (extract, executor.cpp:254-269)."""
    plan = DevicePlan(g, a.m, a.mode, device, 1)
    try:
        Q = a.slabs.shape[0]
        slabs = np.ascontiguousarray(a.slabs)
        sp = ptr_array([slabs[q].ctypes.data for q in range(Q)])
        n, d = g.n, g.d
        vg = np.empty((Q, n + 1, d + 1), np.float64)
        vptr = ptr_array([vg[q].ctypes.data for q in range(Q)])
        dyn = np.empty_like(slabs)
        dptr = ptr_array([dyn[q].ctypes.data for q in range(Q)])
        rep = Report()
        check(lib().pse_plan_run(plan._h, 1, sp, a.total_slots * (d + 1), dptr, vptr, C.byref(rep)))
        a.slabs[...] = dyn
        P = 2 if a.mode == CPLX else 1
        value, grad = _split_vg(vg, P, a.m, n, d)
        out = _report(value, grad, rep)
        out.conv_layer_ms, out.add_layer_ms = plan.layer_ms()
        return out
    finally:
        plan.close()


def _report(value, grad, rep: Report) -> RunReport:
    return RunReport(value, grad, rep.wall_ms, rep.conv_ms, rep.add_ms, rep.scale_ms, rep.h2d_ms, rep.d2h_ms,
                     rep.e2e_ms, int(rep.double_op_count), int(rep.alg_op_count), int(rep.conv_jobs_executed),
                     int(rep.add_jobs_executed), int(rep.kernel_launches), device_ms=rep.device_ms)


def evaluate_packed(n: int, d: int, m: int, mode: str, nvars, indices, exponents, stat: np.ndarray,
                    batch: int = 1, device: int = 0):
    """pse_evaluate on packed arrays. stat: [Q][batch][top][d+1]. Returns
    (vg [Q][batch][n+1][d+1], Report)."""
    check_precision(m)
    Q = (2 if _mode_code(mode) else 1) * m
    nv = np.ascontiguousarray(nvars, np.int32)
    ix = np.ascontiguousarray(indices, np.int32)
    ex = None if exponents is None else np.ascontiguousarray(exponents, np.int32)
    st = np.ascontiguousarray(stat, np.float64)
    vg = np.empty((Q, batch, n + 1, d + 1), np.float64)
    rep = Report()
    check(lib().pse_evaluate(n, d, m, _mode_code(mode), len(nv), ptr(nv), ptr(ix), ptr(ex), batch, ptr(st), ptr(vg),
                             device, C.byref(rep)))
    return vg, rep


def evaluate(p: Polynomial, z: Sequence[np.ndarray], device: int = 0) -> RunReport:
    """evaluate (executor.cpp:271-276): fold exponents, build, stage, run,
    extract -- all on the GPU."""
    _check_inputs(p, z)
    nv, idx, ex = p.shape_arrays()
    st = static_block(p, z)
    Q = st.shape[0]
    vg, rep = evaluate_packed(p.n, p.d, p.m, p.mode, nv, idx, ex, st.reshape(Q, 1, *st.shape[1:]), 1, device)
    value, grad = _split_vg(vg[:, 0], p.a0.shape[0], p.m, p.n, p.d)
    return _report(value, grad, rep)


def eval_direct_packed(n: int, d: int, m: int, mode: str, nvars, indices, exponents, stat: np.ndarray,
                       device: int = 0) -> np.ndarray:
    """eval_direct (oracle_direct.cpp:41-78) on the device -- the independent
    evaluator of `verify` (pse_eval_direct: direct product chains, literal md
    arithmetic). stat: [Q][1+N+n][d+1]; returns vg [Q][n+1][d+1]."""
    check_precision(m)
    Q = (2 if _mode_code(mode) else 1) * m
    nv = np.ascontiguousarray(nvars, np.int32)
    ix = np.ascontiguousarray(indices, np.int32)
    ex = None if exponents is None else np.ascontiguousarray(exponents, np.int32)
    st = np.ascontiguousarray(stat, np.float64)
    vg = np.empty((Q, n + 1, d + 1), np.float64)
    check(lib().pse_eval_direct(n, d, m, _mode_code(mode), len(nv), ptr(nv), ptr(ix), ptr(ex), ptr(st), ptr(vg),
                                device))
    return vg


def within_oracle_guard(d: int, nvars, exponents=None) -> bool:
    nv = np.ascontiguousarray(nvars, np.int32)
    ex = None if exponents is None else np.ascontiguousarray(exponents, np.int32)
    return check(lib().pse_within_oracle_guard(d, len(nv), ptr(nv), ptr(ex))) == 1


# ----------------------------------------------------------------- generator
@dataclass
class Problem:
    id: str
    seed: int
    n: int
    d: int
    m: int
    mode: str
    nvars: np.ndarray
    indices: np.ndarray
    stat: Optional[np.ndarray]  # [Q][1+N+n][d+1]
    exponents: Optional[np.ndarray] = None  # [len(indices)], 0 = none for that monomial

    @property
    def N(self) -> int:
        return len(self.nvars)

    def polynomial(self):
        """(Polynomial, z) views of the packed problem."""
        P = 2 if _mode_code(self.mode) else 1
        s = self.stat.reshape(P, self.m, self.stat.shape[1], self.d + 1)
        mons, pos = [], 0
        for k in range(self.N):
            nk = int(self.nvars[k])
            mons.append(Monomial(s[:, :, 1 + k].copy(), [int(v) for v in self.indices[pos:pos + nk]]))
            pos += nk
        poly = Polynomial(self.n, self.d, s[:, :, 0].copy(), mons)
        z = [s[:, :, 1 + self.N + i].copy() for i in range(self.n)]
        return poly, z


def gen_benchmark(pid: str, d: int, m: int, mode: str = REAL, seed: int = 7, with_static: bool = True) -> Problem:
    n, N, ln = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib().pse_gen_benchmark_size(pid.encode(), C.byref(n), C.byref(N), C.byref(ln)))
    check_precision(m)
    nv = np.empty(N.value, np.int32)
    ix = np.empty(ln.value, np.int32)
    Q = (2 if _mode_code(mode) else 1) * m
    st = np.empty((Q, 1 + N.value + n.value, d + 1), np.float64) if with_static else None
    check(lib().pse_gen_benchmark(pid.encode(), d, m, _mode_code(mode), seed, ptr(nv), ptr(ix), ptr(st)))
    return Problem(pid, seed, n.value, d, m, REAL if _mode_code(mode) == 0 else CPLX, nv, ix, st)


# ----------------------------------------------------------------- problem files
# problem_to_text / problem_from_text / write_problem / read_problem
# (problem_io.hpp:26-30): hexfloat limbs, bit-exact round trip; ParseError
# becomes InvalidArgument("line N: ...").
def _problem_from_handle(h) -> Problem:
    try:
        info = np.zeros(7, np.int64)
        check(lib().pse_problem_info(h, ptr(info)))
        n, N, d, m, mode, seed, ln = (int(v) for v in info)
        buf = C.create_string_buffer(256)
        check(lib().pse_problem_id(h, buf, 256))
        nv, ix, ex = C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)(), C.POINTER(C.c_int32)()
        st = C.POINTER(C.c_double)()
        check(lib().pse_problem_arrays(h, C.byref(nv), C.byref(ix), C.byref(ex), C.byref(st)))
        Q = (2 if mode else 1) * m
        stat = np.ctypeslib.as_array(st, (Q, 1 + N + n, d + 1)).copy()
        exps = np.ctypeslib.as_array(ex, (ln,)).copy() if ex else None
        return Problem(buf.value.decode(), seed, n, d, m, CPLX if mode else REAL,
                       np.ctypeslib.as_array(nv, (N,)).copy(), np.ctypeslib.as_array(ix, (ln,)).copy(), stat, exps)
    finally:
        lib().pse_problem_destroy(h)


def _problem_handle(p: Problem):
    h = C.c_void_p()
    nv = np.ascontiguousarray(p.nvars, np.int32)
    ix = np.ascontiguousarray(p.indices, np.int32)
    ex = None if p.exponents is None else np.ascontiguousarray(p.exponents, np.int32)
    st = np.ascontiguousarray(p.stat, np.float64)
    check(lib().pse_problem_create(p.id.encode(), p.seed, p.n, p.d, p.m, _mode_code(p.mode), p.N, ptr(nv), ptr(ix),
                                   ptr(ex), ptr(st), C.byref(h)))
    return h


def problem_from_text(text: str) -> Problem:
    h = C.c_void_p()
    check(lib().pse_problem_parse(text.encode(), C.byref(h)))
    return _problem_from_handle(h)


def problem_to_text(p: Problem) -> str:
    h = _problem_handle(p)
    try:
        n = C.c_size_t()
        check(lib().pse_problem_text(h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(lib().pse_problem_text(h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()
    finally:
        lib().pse_problem_destroy(h)


def read_problem(path: str) -> Problem:
    h = C.c_void_p()
    check(lib().pse_problem_read(path.encode(), C.byref(h)))
    return _problem_from_handle(h)


def write_problem(path: str, p: Problem) -> None:
    h = _problem_handle(p)
    try:
        check(lib().pse_problem_write(h, path.encode()))
    finally:
        lib().pse_problem_destroy(h)


# ----------------------------------------------------------------- primitives
def md_apply(op: str, x: np.ndarray, y: np.ndarray, impl: str = "fast", device: int = 0) -> np.ndarray:
    """Elementwise md_add/md_sub/md_mul on the GPU over [count][m] arrays."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    count, m = x.shape
    out = np.empty_like(x)
    check(lib().pse_md_apply({"add": 0, "sub": 1, "mul": 2}[op], m, {"fast": 0, "lit": 1}[impl], count, ptr(x),
                             ptr(y), ptr(out), device))
    return out


def series_conv(x: np.ndarray, y: np.ndarray, mode: str = REAL, device: int = 0) -> np.ndarray:
    """conv (pseries.cpp:37-64) of count pairs: x, y [count][P][m][d+1]."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    count, P, m, d1 = x.shape
    z = np.empty_like(x)
    check(lib().pse_series_conv(d1 - 1, m, _mode_code(mode), count, ptr(x), ptr(y), ptr(z), device))
    return z


def series_add(x: np.ndarray, y: np.ndarray, mode: str = REAL, device: int = 0) -> np.ndarray:
    """series_add (pseries.cpp:66-74) of count pairs: x, y [count][P][m][d+1]."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    count, P, m, d1 = x.shape
    z = np.empty_like(x)
    check(lib().pse_series_add(d1 - 1, m, _mode_code(mode), count, ptr(x), ptr(y), ptr(z), device))
    return z


def series_scale_int(x: np.ndarray, factor: int, mode: str = REAL, device: int = 0) -> np.ndarray:
    """series_scale_int (pseries.cpp:85-93) of count series: x [count][P][m][d+1]."""
    x = np.ascontiguousarray(x, np.float64)
    count, P, m, d1 = x.shape
    z = np.empty_like(x)
    check(lib().pse_series_scale_int(d1 - 1, m, _mode_code(mode), count, ptr(x), int(factor), ptr(z), device))
    return z


def device_info(device: int = 0):
    out = np.zeros(4, np.int64)
    check(lib().pse_device_info(device, ptr(out)))
    return dict(sms=int(out[0]), clock_khz=int(out[1]), cc=int(out[2]), count=int(out[3]))


def fp64_peak(device: int = 0):
    """Measured FP64 issue rate: dict(dadd=lane-ops/s, dfma=lane-ops/s)."""
    out = np.zeros(4, np.float64)
    check(lib().pse_fp64_peak(device, ptr(out)))
    return dict(dadd=float(out[0]), dfma=float(out[1]), blocks=int(out[2]), ms=float(out[3]))
