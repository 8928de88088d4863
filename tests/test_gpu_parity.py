"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle,
bit for bit. Mirrors the reference's own assertions:
  engine == eval_direct on positive-integer instances  (test_executor.cpp:148-179)
  device == run_sequential on p1, d in {8,31}, m in {1,2,4} (acceptance.cpp:163-189)
  md identities bitwise (test_multidouble.cpp:148-163)
plus bitwise equality with the oracle on full-precision instances for every
precision level, on the C1 correctness configuration, and through the
batched multi-point path."""
import numpy as np
import pytest

import pyoracle as po
from instances import assert_bitwise, int_instance, md_instance

pe = pytest.importorskip("paper_2101_10881_b200")

pytestmark = pytest.mark.gpu
LEVELS = [1, 2, 3, 4, 5, 8, 10]


@pytest.fixture(params=["fused", "split", "band", "flow", "flow32", "cta", "ctl"])
def conv_path(request, monkeypatch):
    """Run an engine test through the fused conv kernel (one thread per
    coefficient pair), through the split path (products in parallel, then
    the accumulation chains), through the banded wavefront (chains cut into
    band x segment tasks, scheduled across layers, one launch per wave) and
    through its dataflow form (one persistent launch, per-task completion
    flags; 16- and 32-wide bands) and the CTA-local dataflow (one block per
    job group, shared-memory flags; where a group's flags do not fit next to
    the lanes -- M >= 8 -- the global dataflow runs) and the CTA-local layered
    walk (one block per job group, its layers in order). The planner reads
    PSE_CONV_MODE and PSE_SPLIT_THRESHOLD when a plan is created: 0 forces
    fused, a huge value forces split."""
    if request.param in ("cta", "ctl"):
        monkeypatch.setenv("PSE_CONV_MODE", request.param)
    elif request.param in ("band", "flow", "flow32"):
        # waves use 32-wide bands, the dataflow kernel 16 (flow32: 32)
        monkeypatch.setenv("PSE_CONV_MODE", request.param[:4])
        if request.param == "flow32":
            monkeypatch.setenv("PSE_BAND_W", "32")
    else:
        monkeypatch.setenv("PSE_CONV_MODE", "layer")
        monkeypatch.setenv("PSE_SPLIT_THRESHOLD", "0" if request.param == "fused" else str(1 << 60))
    return request.param


def dev_eval(p: po.Problem, batch_stat=None):
    """evaluate() on the device for one problem; returns vg [P][m][n+1][d+1]."""
    Q = p.P * p.m
    st = p.stat.reshape(Q, 1, *p.stat.shape[2:]) if batch_stat is None else batch_stat
    vg, rep = pe.evaluate_packed(p.n, p.d, p.m, "cplx" if p.cplx else "real", p.nvars, p.idx, p.exps, st,
                                 st.shape[1])
    return vg, rep


# ---------------------------------------------------------------- md ops
@pytest.mark.parametrize("m", LEVELS)
@pytest.mark.parametrize("impl", ["fast", "lit"])
def test_md_ops_bitwise_random(m, impl):
    x = po.random_md(1000 + m, m, 200_000)
    y = po.random_md(2000 + m, m, 200_000)
    for op in ("add", "sub", "mul"):
        assert_bitwise(pe.md_apply(op, x, y, impl), po.md_op(op, x, y), f"{op} m={m} {impl}")


@pytest.mark.parametrize("m", LEVELS)
def test_md_ops_bitwise_edge_cases(m):
    rng = np.random.default_rng(m)
    base = po.random_md(77 + m, m, 64)
    specials = []
    z = np.zeros(m)
    nz = -np.zeros(m)
    one = np.zeros(m)
    one[0] = 1.0
    specials += [z, nz, one, -one]
    for v in base[:16]:
        specials += [v, -v]
        w = v.copy()
        w[1:] = 0.0
        specials.append(w)  # leading limb only
        if m > 1:
            u = v.copy()
            u[-1] = -0.0
            specials.append(u)
    ints = np.zeros((32, m))
    ints[:, 0] = rng.integers(-50, 50, 32)
    specials += list(ints)
    S = np.array(specials)
    X = np.repeat(S, len(S), 0)
    Y = np.tile(S, (len(S), 1))
    for op in ("add", "sub", "mul"):
        assert_bitwise(pe.md_apply(op, X, Y, "fast"), po.md_op(op, X, Y), f"{op} m={m} edge")


@pytest.mark.parametrize("m", LEVELS)
def test_md_identities(m):
    """x+0, x-0, x*1 bitwise x; x*0 all zeros (test_multidouble.cpp:148-163)."""
    x = po.random_md(4000 + m, m, 300)
    zero = np.zeros_like(x)
    one = np.zeros_like(x)
    one[:, 0] = 1.0
    assert_bitwise(pe.md_apply("add", x, zero), x, "x+0")
    assert_bitwise(pe.md_apply("sub", x, zero), x, "x-0")
    assert_bitwise(pe.md_apply("mul", x, one), x, "x*1")
    assert (pe.md_apply("mul", x, zero) == 0.0).all()


# ---------------------------------------------------------------- series conv
@pytest.mark.parametrize("m", LEVELS)
@pytest.mark.parametrize("cplx", [False, True])
def test_series_conv_bitwise(m, cplx):
    rng = np.random.default_rng(10 * m + cplx)
    P = 2 if cplx else 1
    for d in (0, 1, 2, 7, 16, 33):
        cnt = 5
        x = po.random_md(int(rng.integers(1, 2**60)), m, cnt * P * (d + 1)).reshape(cnt, P, d + 1, m).transpose(0, 1, 3, 2).copy()
        y = po.random_md(int(rng.integers(1, 2**60)), m, cnt * P * (d + 1)).reshape(cnt, P, d + 1, m).transpose(0, 1, 3, 2).copy()
        z = pe.series_conv(x, y, "cplx" if cplx else "real")
        for c in range(cnt):
            assert_bitwise(z[c], po.series_conv(x[c], y[c], cplx), f"conv d={d} m={m} c={c}")


@pytest.mark.parametrize("m", LEVELS)
@pytest.mark.parametrize("cplx", [False, True])
def test_series_add_and_scale_bitwise(m, cplx):
    """series_add / series_scale_int (pseries.cpp:66-93) over the C ABI equal
    the oracle's md_add / md_mul by md_from_double(c) per coefficient."""
    rng = np.random.default_rng(20 * m + cplx)
    P, d, cnt = (2 if cplx else 1), 17, 4
    x = po.random_md(int(rng.integers(1, 2**60)), m, cnt * P * (d + 1)).reshape(cnt, P, d + 1, m).transpose(0, 1, 3, 2).copy()
    y = po.random_md(int(rng.integers(1, 2**60)), m, cnt * P * (d + 1)).reshape(cnt, P, d + 1, m).transpose(0, 1, 3, 2).copy()
    mode = "cplx" if cplx else "real"
    flat = lambda a: a.transpose(0, 1, 3, 2).reshape(-1, m).copy()  # [count*P*(d+1)][m]
    z = pe.series_add(x, y, mode)
    assert_bitwise(flat(z), po.md_op("add", flat(x), flat(y)), f"series_add m={m}")
    for c in (3, -7, 0, 1 << 20):
        cm = np.zeros_like(flat(x))
        cm[:, 0] = float(c)
        z = pe.series_scale_int(x, c, mode)
        assert_bitwise(flat(z), po.md_op("mul", flat(x), cm), f"series_scale_int c={c} m={m}")


# ---------------------------------------------------------------- whole engine
def test_c1_bitwise_vs_reference_engine(conv_path):
    """C1: p1, d=15, m=2, seed 7 -- value, all 16 gradients and the whole
    dynamic arena equal run_sequential bit for bit."""
    p = po.gen_benchmark("p1", 15, 2, seed=7)
    ref_vg, ref_dyn = po.evaluate(p, "ref" if po.has_ref() else "port", want_dyn=True)
    pr = pe.gen_benchmark("p1", 15, 2, seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    plan = pe.DevicePlan(g, 2, "real", 0, 1)
    vg, dyn, rep = plan.run(pr.stat, 1, want_dyn=True)
    assert_bitwise(vg[:, 0], ref_vg.reshape(2, 17, 16), "C1 value/gradients")
    assert_bitwise(dyn[:, 0], ref_dyn.reshape(2, -1, 16), "C1 arena")
    assert rep.conv_jobs_executed == 16380 and rep.add_jobs_executed == 9084
    assert rep.double_op_count == po.flop_count(p, 39, 94)


@pytest.mark.parametrize("d", [8, 31])
@pytest.mark.parametrize("m", [1, 2, 4])
def test_p1_bitwise_vs_sequential(d, m, conv_path):
    """acceptance criterion 6 (acceptance.cpp:163-189) with the device engine."""
    p = po.gen_benchmark("p1", d, m, seed=7)
    ref = po.evaluate(p, "port")
    vg, _ = dev_eval(p)
    assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"p1 d={d} m={m}")


@pytest.mark.parametrize("pid", ["p1", "p2", "p3"])
@pytest.mark.parametrize("d", [0, 1, 2, 3, 5])
def test_m1_small_degrees_default_path(pid, d):
    """m=1 through the planner's default (the CTA-local layer walk: register
    blocks of three chains, the last block partly past d) at degrees whose
    chains are shorter than one block"""
    p = po.gen_benchmark(pid, d, 1, seed=7)
    ref = po.evaluate(p, "port")
    vg, _ = dev_eval(p)
    assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"{pid} d={d} m=1")


@pytest.mark.parametrize("pid,d,m", [("p2", 3, 2), ("p3", 3, 2), ("p2", 8, 10), ("p3", 2, 10)])
def test_p2_p3_bitwise(pid, d, m, conv_path):
    p = po.gen_benchmark(pid, d, m, seed=7)
    ref = po.evaluate(p, "port")
    vg, _ = dev_eval(p)
    assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"{pid} d={d} m={m}")


def test_integer_instances_equal_direct_oracle(conv_path):
    """200 positive-integer instances (half with exponents): device ==
    eval_direct bitwise (test_executor.cpp:148-159, acceptance criterion 5)."""
    rng = np.random.default_rng(506)
    for it in range(200):
        p = int_instance(rng, it % 2 == 1)
        ref = po.eval_direct(p)
        vg, _ = dev_eval(p)
        assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"int instance {it}")


def test_complex_integer_instances_equal_direct_oracle(conv_path):
    rng = np.random.default_rng(507)
    for it in range(40):
        p = int_instance(rng, False, cplx=True)
        ref = po.eval_direct(p)
        vg, _ = dev_eval(p)
        assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"complex int instance {it}")


@pytest.mark.parametrize("m", LEVELS)
@pytest.mark.parametrize("cplx", [False, True])
def test_md_instances_bitwise_vs_oracle(m, cplx, conv_path):
    rng = np.random.default_rng(900 + m + 50 * cplx)
    for it in range(12):
        p = md_instance(rng, m, cplx, with_exponents=it % 3 == 0)
        ref = po.evaluate(p, "port")
        vg, _ = dev_eval(p)
        assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"md instance m={m} cplx={cplx} it={it}")


@pytest.mark.parametrize("pid,d,m", [("p2", 40, 2), ("p2", 70, 1), ("p1", 66, 2)])
def test_multiband_graphs_bitwise(pid, d, m, conv_path):
    """Degrees past one band (32 coefficients): the banded path cuts every
    chain into segments and carries partial sums between waves."""
    p = po.gen_benchmark(pid, d, m, seed=7)
    ref = po.evaluate(p, "port")
    vg, _ = dev_eval(p)
    assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"{pid} d={d} m={m}")


@pytest.mark.parametrize("m", LEVELS)
@pytest.mark.parametrize("cplx", [False, True])
def test_multiband_md_instances(m, cplx, conv_path):
    rng = np.random.default_rng(1900 + m + 50 * cplx)
    for it in range(4):
        p = md_instance(rng, m, cplx, nmax=5, Nmax=5, dmin=33, dmax=100, with_exponents=it % 2 == 1)
        ref = po.evaluate(p, "port")
        vg, _ = dev_eval(p)
        assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"md instance m={m} cplx={cplx} d={p.d} it={it}")


@pytest.mark.parametrize("m", [4, 1])
def test_batched_points_equal_single_points(conv_path, m):
    """one launch per layer across a batch of points == each point alone."""
    rng = np.random.default_rng(42)
    base = po.gen_benchmark("p1", 12, m, seed=7)
    B = 5
    Q = base.P * base.m
    top = base.stat.shape[2]
    stat = np.empty((Q, B, top, 13))
    refs = []
    for b in range(B):
        zb = po.gen_benchmark("p1", 12, m, seed=1000 + b)
        s = base.stat.copy()
        s[:, :, 1 + base.N:] = zb.stat[:, :, 1 + base.N:]  # point b's inputs
        stat[:, b] = s.reshape(Q, top, 13)
        q = po.Problem(base.n, base.d, base.m, False, base.nvars, base.idx, None, s)
        refs.append(po.evaluate(q, "port"))
    vg, rep = dev_eval(base, stat)
    for b in range(B):
        assert_bitwise(vg[:, b].reshape(refs[b].shape), refs[b], f"point {b}")
    assert rep.batch == B


def test_errors_are_invalid_argument():
    with pytest.raises(pe.InvalidArgument):
        pe.evaluate_packed(2, 3, 7, "real", [1], [1], None, np.zeros((7, 1, 4, 4)))
    with pytest.raises(pe.InvalidArgument):
        pe.evaluate_packed(2, 3, 2, "real", [2], [2, 1], None, np.zeros((2, 1, 4, 4)))


def _p2h(p: po.Problem) -> po.Problem:
    """C3': p2's even cyclic windows (bench.py make_static)."""
    keep = np.arange(0, p.N, 2)
    starts = np.concatenate([[0], np.cumsum(p.nvars)])
    idx = np.concatenate([p.idx[starts[k]:starts[k + 1]] for k in keep]).astype(np.int32)
    stat = np.concatenate([p.stat[:, :, :1], p.stat[:, :, 1 + keep], p.stat[:, :, 1 + p.N:]], axis=2)
    return po.Problem(p.n, p.d, p.m, p.cplx, p.nvars[keep].copy(), idx, None, np.ascontiguousarray(stat), "p2h")


@pytest.mark.parametrize("cfg,pid,m", [("C2", "p1", 10), ("C3", "p2", 10), ("C3'", "p2h", 10), ("C4", "p3", 10),
                                       ("C3 m=1", "p2", 1), ("C3 m=2", "p2", 2), ("C3 m=5", "p2", 5),
                                       ("C1", "p1", 2)])
def test_benchmark_configs_full_size_bitwise_vs_reference_engine(cfg, pid, m):
    """The BASELINE configurations at full size (d=152, seed 7; C1 at d=15)
    through the conv path the planner picks for them (layered/hybrid for C2
    and C4, dataflow for C3 and C3', the CTA-local layer walk for C3 at m=1,
    layered for C1): value and every gradient series equal the reference
    engine's run_parallel (oracle/_ref, the reference's own sources) bit for
    bit."""
    import os

    if not po.has_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    p = po.gen_benchmark("p2" if pid == "p2h" else pid, 15 if cfg == "C1" else 152, m, seed=7)
    if pid == "p2h":
        p = _p2h(p)
    ref = po.evaluate(p, "ref", workers=os.cpu_count() or 1)
    g = pe.build_jobgraph_shape(p.n, p.d, p.nvars, p.idx)
    plan = pe.DevicePlan(g, m, "real", 0, 1)
    vg, _, rep = plan.run(p.stat.reshape(p.P * m, *p.stat.shape[2:]), 1)
    assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"{cfg}: {pid} d=152 m={m} ({plan.conv_path(1)})")


def _c5_wave_as_benched(d, m, total, first, batch):
    """C5 exactly as bench.py stages it: the static blocks of points
    [0, total) (coefficients of seed 7, point b's z from seed 1000+b,
    bench.make_static) resident in HBM as one CUDA tensor, points
    [first, first+batch) staged into the plan by DevicePlan.upload_ptr (a D2D
    copy out of the middle of the buffer), then the captured-graph replay
    the timed steps use. Returns (stat [Q][total][top][d+1], plan, vg of the
    wave)."""
    import torch

    import bench

    n, N, nvars, idx, stat = bench.make_static("p2h", d, m, range(total))
    g = pe.build_jobgraph_shape(n, d, nvars, idx)
    plan = pe.DevicePlan(g, m, "real", 0, batch)
    stat_dev = torch.from_numpy(np.ascontiguousarray(stat)).to("cuda:0")
    torch.cuda.synchronize()
    plan.upload_ptr(stat_dev.data_ptr(), batch, total=total, first=first)
    plan.execute(batch, detail=False)
    vg, _ = plan.download(batch)
    return (n, N, nvars, idx, stat), plan, vg


@pytest.mark.timeout(1200)
def test_c5_wave_as_benched_bitwise():
    """BASELINE C5 (p2h, d=152, m=10, point b's inputs from seed 1000+b,
    gen.cpp:50-71) through the bench's own staging path: a 16-point wave
    taken from the middle of a 40-point device buffer (first=9, total=40)
    equals each point evaluated alone on the device, and points of the wave
    equal the reference engine (oracle/_ref run_parallel) bit for bit."""
    import os

    d, m, total, first, batch = 152, 10, 40, 9, 16
    (n, N, nvars, idx, stat), plan, vg = _c5_wave_as_benched(d, m, total, first, batch)
    assert plan.conv_path(batch) in ("layered", "hybrid", "dataflow")
    g = plan.graph
    single = pe.DevicePlan(g, m, "real", 0, 1)
    for b in range(batch):
        one, _, _ = single.run(np.ascontiguousarray(stat[:, first + b]), 1)
        assert_bitwise(vg[:, b], one[:, 0], f"C5 wave point {first + b} vs single-point run")
    if not po.has_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    for b in (0, batch - 1):
        p = po.Problem(n, d, m, False, nvars, idx, None, stat[:, first + b].reshape(1, m, -1, d + 1))
        ref = po.evaluate(p, "ref", workers=os.cpu_count() or 1)
        assert_bitwise(vg[:, b].reshape(ref.shape), ref, f"C5 point {first + b} vs reference engine")


@pytest.mark.timeout(1200)
def test_c5_grid_of_128_points_bitwise():
    """The grid size C5 runs at (waves of 128 points in one launch per
    layer), on a smaller degree: a 128-point wave at offset 3 of a 140-point
    device buffer equals the C oracle point by point."""
    d, m, total, first, batch = 20, 3, 140, 3, 128
    (n, N, nvars, idx, stat), plan, vg = _c5_wave_as_benched(d, m, total, first, batch)
    for b in list(range(0, batch, 9)) + [batch - 1]:
        p = po.Problem(n, d, m, False, nvars, idx, None, stat[:, first + b].reshape(1, m, -1, d + 1))
        ref = po.evaluate(p, "port")
        assert_bitwise(vg[:, b].reshape(ref.shape), ref, f"128-point wave, point {first + b}")


@pytest.mark.parametrize("pid,d,m", [("p1", 64, 4), ("p2", 40, 2), ("p1", 152, 10)])
def test_complex_benchmark_graphs_bitwise_vs_reference_engine(pid, d, m):
    """Complex mode (separate re/im slabs, the complex conv of pseries.cpp:49-59)
    on the benchmark graphs, up to C2's full size, against the reference
    engine."""
    import os

    if not po.has_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    p = po.gen_benchmark(pid, d, m, cplx=True, seed=7)
    ref = po.evaluate(p, "ref", workers=os.cpu_count() or 1)
    g = pe.build_jobgraph_shape(p.n, p.d, p.nvars, p.idx)
    plan = pe.DevicePlan(g, m, "cplx", 0, 1)
    vg, _, _ = plan.run(p.stat.reshape(p.P * m, *p.stat.shape[2:]), 1)
    assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"complex {pid} d={d} m={m} ({plan.conv_path(1)})")


@pytest.mark.parametrize("m", [2, 10])
def test_exponents_at_full_degree_bitwise(m):
    """Monomials with exponents (device fold_exponents prologue) at d=152."""
    rng = np.random.default_rng(4242 + m)
    for it in range(3):
        p = md_instance(rng, m, False, nmax=6, Nmax=8, dmin=152, dmax=152, with_exponents=True)
        ref = po.evaluate(p, "port")
        vg, _ = dev_eval(p)
        assert_bitwise(vg[:, 0].reshape(ref.shape), ref, f"exponents m={m} it={it}")


def test_reference_binding_drop_in():
    """include/pse_b200_pseval.hpp compiled against the unmodified reference
    sources: run_device == run_sequential bit for bit on the reference's own
    DataArray (oracle/integration_check.cpp; built where /root/reference was
    available)."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(po.__file__), "_ref", "integration_check")
    if not os.path.exists(exe):
        pytest.skip("integration_check not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK: 4/4" in r.stdout
    assert "OK: RunReport per-layer timings" in r.stdout, r.stdout


@pytest.mark.parametrize("pid,d,m,nranks", [("p1", 15, 2, 2), ("p1", 8, 4, 3), ("p3", 4, 2, 4), ("p2", 3, 3, 2),
                                             ("p1", 15, 1, 3), ("p3", 4, 1, 4)])
def test_monomial_sharding_is_bit_exact(pid, d, m, nranks):
    """One polynomial sharded over nranks plans (here all on device 0): each
    runs its monomials' conv jobs, the term blocks are exchanged, each runs the
    exact addition tree -- every rank's result equals one device's, bit for
    bit, and the reference's."""
    import torch

    pr = pe.gen_benchmark(pid, d, m, seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    full = pe.DevicePlan(g, m, "real", 0, 1)
    ref_vg, _, _ = full.run(pr.stat, 1)
    plans = [pe.DevicePlan(g, m, "real", 0, 1, rank=r, nranks=nranks) for r in range(nranks)]
    width = max(1, max(plans[0].exchange_words(r) for r in range(nranks)))
    blocks = []
    for p in plans:
        p.upload(pr.stat, 1)
        p.execute(1, detail=True)
        buf = torch.zeros(width, dtype=torch.float64, device="cuda:0")
        torch.cuda.synchronize()  # the fill (torch's stream) before pack (the plan's stream)
        p.pack(buf.data_ptr())
        blocks.append(buf)
    assert sum(plans[0].exchange_words(r) for r in range(nranks)) > 0
    for p in plans:
        for r in range(nranks):
            p.unpack(r, blocks[r].data_ptr())
        rep = p.finish(1)
        assert rep.kernel_launches > 0
        vg, _ = p.download(1)
        assert_bitwise(vg, ref_vg, f"{pid} rank {p.rank}/{nranks}")
    want = po.evaluate(po.gen_benchmark(pid, d, m, seed=7), "port")
    assert_bitwise(ref_vg[:, 0].reshape(want.shape), want, "vs oracle")


@pytest.mark.parametrize("pid,d,m,nranks", [("p1", 15, 2, 2), ("p3", 4, 2, 4), ("p2", 40, 3, 3), ("p2", 40, 1, 3)])
def test_monomial_sharding_peer_gather_is_bit_exact(pid, d, m, nranks):
    """The same sharding with the exchange done by pse_plan_gather_peers: each
    rank copies the slots the other ranks produced straight out of their
    arenas (here plans of one process on one device)."""
    pr = pe.gen_benchmark(pid, d, m, seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    full = pe.DevicePlan(g, m, "real", 0, 1)
    ref_vg, _, _ = full.run(pr.stat, 1)
    plans = [pe.DevicePlan(g, m, "real", 0, 1, rank=r, nranks=nranks) for r in range(nranks)]
    for p in plans:
        for q in plans:
            if q is not p:
                p.set_peer(q.rank, q)
        p.upload(pr.stat, 1)
        p.execute(1, detail=True)
    for p in plans:
        p.gather_peers(1)
    for p in plans:
        p.finish(1)
        vg, _ = p.download(1)
        assert_bitwise(vg, ref_vg, f"{pid} rank {p.rank}/{nranks} (peer gather)")


def _ipc_worker(rank, world, port, outdir):
    import os
    import sys

    import torch

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import paper_2101_10881_b200 as pe2
    from paper_2101_10881_b200 import dist as DD

    dist = DD.init("gloo")
    torch.cuda.set_device(0)
    pr = pe2.gen_benchmark("p1", 15, 2, seed=7)
    g = pe2.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    plan = pe2.DevicePlan(g, 2, "real", 0, 1, rank=rank, nranks=world)
    assert DD.connect_peers(plan)
    plan.upload(pr.stat, 1)
    for _ in range(2):  # twice: the barriers also order consecutive evaluations
        DD.evaluate_sharded(plan, 1, p2p=True)
    vg, _ = plan.download(1)
    np.save(os.path.join(outdir, f"vg{rank}.npy"), vg)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_monomial_sharding_ipc_processes_bit_exact(tmp_path):
    """Two processes (ranks) sharing the GPU: arenas mapped through CUDA IPC
    handles exchanged over gloo, the peer gather between barriers; both
    ranks' results equal one device's bit for bit."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_ipc_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    pr = pe.gen_benchmark("p1", 15, 2, seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    ref_vg, _, _ = pe.DevicePlan(g, 2, "real", 0, 1).run(pr.stat, 1)
    for r in range(2):
        assert_bitwise(np.load(tmp_path / f"vg{r}.npy"), ref_vg, f"ipc rank {r}")


def test_plan_reused_across_batch_sizes():
    """One plan run at batch 1, 3 and 1 again through its captured CUDA
    graphs (the dataflow path keeps per-batch task tables and flags): every
    run equals the single-point evaluation bit for bit."""
    base = po.gen_benchmark("p2", 40, 2, seed=7)
    Q = base.P * base.m
    top = base.stat.shape[2]
    stat = np.empty((Q, 3, top, 41))
    refs = []
    for b in range(3):
        zb = po.gen_benchmark("p2", 40, 2, seed=1000 + b)
        st = base.stat.copy()
        st[:, :, 1 + base.N:] = zb.stat[:, :, 1 + base.N:]
        stat[:, b] = st.reshape(Q, top, 41)
        refs.append(po.evaluate(po.Problem(base.n, base.d, base.m, False, base.nvars, base.idx, None, st), "port"))
    g = pe.build_jobgraph_shape(base.n, base.d, base.nvars, base.idx)
    plan = pe.DevicePlan(g, 2, "real", 0, 3)
    for batch in (1, 3, 1, 3):
        plan.upload(np.ascontiguousarray(stat[:, :batch]), batch)
        plan.execute(batch, detail=False)
        vg, _ = plan.download(batch)
        for b in range(batch):
            assert_bitwise(vg[:, b].reshape(refs[b].shape), refs[b], f"batch {batch} point {b} ({plan.conv_path(batch)})")


def test_cli_verify_and_bench(tmp_path):
    """pseval_b200 verify / bench (the reference CLI's subcommands over the
    device engine): verify compares the layered fused and split convolutions,
    the dataflow and banded-wave schedules, the two CTA-local forms, the
    planner's path and a batch of points bit for bit, and the engine with the independent device evaluator
    within the reference's tolerance (pseval.cpp:97-118)."""
    import os
    import subprocess

    cli = os.path.join(os.path.dirname(pe.LIB_PATH), "pseval_b200")
    for args in (["verify", "p1", "--degree", "8", "--precision", "4", "--oracle", "on"],
                 ["verify", "p3", "--degree", "5", "--precision", "2", "--mode", "complex", "--oracle", "on"],
                 ["verify", "p2", "--degree", "20", "--precision", "3", "--oracle", "on"]):
        r = subprocess.run([cli, *args], capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "verify: PASS" in r.stdout, r.stdout + r.stderr
        assert r.stdout.count("bitwise equal") == 7, r.stdout
        assert "oracle: independent device evaluator" in r.stdout and ": ok" in r.stdout, r.stdout
    path = str(tmp_path / "p2.txt")
    assert subprocess.run([cli, "gen", "p2", path, "--degree", "3", "--precision", "3"]).returncode == 0
    r = subprocess.run([cli, "verify", path], capture_output=True, text=True, timeout=600)
    assert "verify: PASS" in r.stdout, r.stdout + r.stderr
    csv = str(tmp_path / "b.csv")
    r = subprocess.run([cli, "bench", "p1", "--degree", "8", "15", "--precision", "2", "--repeats", "2", "--csv", csv],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert "| p1 | 15 | 2 | real |" in r.stdout
    rows = open(csv).read().strip().split("\n")
    assert rows[0].startswith("id,d,m,mode,workers") and len(rows) == 3


@pytest.mark.parametrize("which,line", [("split", "layered fused vs layered split convolutions: MISMATCH"),
                                        ("flow", "dataflow (banded, one persistent launch) vs layered: MISMATCH"),
                                        ("band", "banded waves vs layered: MISMATCH"),
                                        ("cta", "CTA-local dataflow vs layered: MISMATCH"),
                                        ("ctl", "CTA-local layers vs layered: MISMATCH"),
                                        ("oracle", "max coefficient discrepancy")])
def test_cli_verify_fails_on_a_broken_path(which, line):
    """verify is not vacuous: a one-ulp change in one path's result (or a
    1e-6 relative change in every path, against the independent evaluator)
    turns it into FAIL"""
    import os
    import subprocess

    cli = os.path.join(os.path.dirname(pe.LIB_PATH), "pseval_b200")
    env = dict(os.environ, PSE_VERIFY_PERTURB=which)
    r = subprocess.run([cli, "verify", "p1", "--degree", "8", "--precision", "4", "--oracle", "on"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 1 and "verify: FAIL" in r.stdout, r.stdout + r.stderr
    assert line in r.stdout, r.stdout
    if which == "oracle":
        assert "MISMATCH" in r.stdout.split("oracle:")[1]


def test_cli_verify_refuses_instances_beyond_the_guard():
    """--oracle on past within_oracle_guard (oracle_direct.cpp:32-39): refused, exit code 2"""
    import os
    import subprocess

    cli = os.path.join(os.path.dirname(pe.LIB_PATH), "pseval_b200")
    r = subprocess.run([cli, "verify", "p3", "--degree", "60", "--precision", "1", "--oracle", "on"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 2 and "refused" in r.stdout, r.stdout + r.stderr


def test_device_eval_direct_equals_reference_eval_direct():
    """pse_eval_direct (the independent evaluator of verify: direct product
    chains, literal md arithmetic) equals the reference's own eval_direct
    (oracle_direct.cpp:41-78) bit for bit -- integer and full-precision
    instances, real and complex, with exponents"""
    lib = "ref" if po.has_ref() else "port"
    rng = np.random.default_rng(2024)
    for it in range(40):
        p = int_instance(rng, it % 2 == 1, cplx=it % 4 == 3)
        ref = po.eval_direct(p, lib)
        vg = pe.eval_direct_packed(p.n, p.d, p.m, "cplx" if p.cplx else "real", p.nvars, p.idx, p.exps,
                                   p.stat.reshape(p.P * p.m, *p.stat.shape[2:]))
        assert_bitwise(vg.reshape(ref.shape), ref, f"int instance {it}")
    for m in LEVELS:
        for cplx in (False, True):
            p = md_instance(rng, m, cplx, with_exponents=True)
            if not pe.within_oracle_guard(p.d, p.nvars, p.exps):
                continue
            ref = po.eval_direct(p, lib)
            vg = pe.eval_direct_packed(p.n, p.d, p.m, "cplx" if cplx else "real", p.nvars, p.idx, p.exps,
                                       p.stat.reshape(p.P * m, *p.stat.shape[2:]))
            assert_bitwise(vg.reshape(ref.shape), ref, f"md instance m={m} cplx={cplx}")


def test_slot_rewritten_in_a_later_layer_stays_exact():
    """validate() (jobgraph.cpp:273-336) accepts a dynamic slot written again
    in a later conv layer. The banded/dataflow schedule assumes one producer
    per slot, so the planner keeps such graphs on the layered path (with the
    dataflow path forced, too). The result equals the same graph with the
    rewrite sent to a fresh slot and the addition stage reading that slot."""
    import os

    pr = pe.gen_benchmark("p1", 6, 2, seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    top = 1 + g.N + g.n
    F = int(next(s for s in g.add_src if s >= top))  # a dynamic term slot the addition stage reads
    z1, z2 = top - g.n, top - g.n + 1  # two input slots
    off = list(g.conv_layer_off) + [g.conv_layer_off[-1] + 1]

    def graph_with_rewrite(out, total, add_src, add_dst, value_slot, grads):
        return pe.GraphArrays(g.n, g.N, g.d, total, value_slot, grads, g.multipliers, off,
                              list(g.conv_in1) + [z1], list(g.conv_in2) + [z2], list(g.conv_out) + [out],
                              list(g.conv_copy) + [0], g.add_layer_off, add_src, add_dst)

    multi = graph_with_rewrite(F, g.total_slots, g.add_src, g.add_dst, g.value_slot, g.gradient_slots)
    assert pe.validate(multi)[0]
    Fp = g.total_slots  # the renamed twin: the rewrite goes to a fresh slot
    ren = lambda a: [Fp if int(s) == F else int(s) for s in a]
    renamed = graph_with_rewrite(Fp, g.total_slots + 1, ren(g.add_src), ren(g.add_dst),
                                 ren([g.value_slot])[0], ren(g.gradient_slots))
    assert pe.validate(renamed)[0]
    st = pr.stat.reshape(2, 1, *pr.stat.shape[1:])[:, 0]
    want, _, _ = pe.DevicePlan(renamed, 2, "real", 0, 1).run(st, 1)
    for mode in ("", "flow"):
        if mode:
            os.environ["PSE_CONV_MODE"] = mode
        try:
            plan = pe.DevicePlan(multi, 2, "real", 0, 1)
            assert plan.conv_path(1) == "layered"
            got, _, _ = plan.run(st, 1)
        finally:
            os.environ.pop("PSE_CONV_MODE", None)
        assert_bitwise(got, want, f"rewritten slot (PSE_CONV_MODE={mode or 'auto'})")


@pytest.mark.parametrize("mode", ["", "layer", "flow"])
def test_run_report_per_layer_times(mode, monkeypatch):
    """RunReport's per-phase lists (executor.hpp:31-43, executor.cpp:154-157)
    from the kernels' own stamps, through run_device: one entry per conv and
    per add layer, non-negative, summing to conv_ms / add_ms, and with the
    scale phase to wall_ms; the graph-replay path reports them too."""
    if mode:
        monkeypatch.setenv("PSE_CONV_MODE", mode)
    pr = pe.gen_benchmark("p1", 40, 3, seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    poly, z = pr.polynomial()
    a = pe.stage(poly, z)
    r = pe.run_device(g, a)
    assert len(r.conv_layer_ms) == len(g.conv_layer_sizes()) and len(r.add_layer_ms) == len(g.add_layer_sizes())
    assert min(r.conv_layer_ms) >= 0 and min(r.add_layer_ms) >= 0
    assert r.conv_ms > 0 and r.add_ms > 0
    assert abs(sum(r.conv_layer_ms) - r.conv_ms) <= 1e-9 + 1e-6 * r.conv_ms
    assert abs(sum(r.add_layer_ms) - r.add_ms) <= 1e-9 + 1e-6 * r.add_ms
    assert abs(r.conv_ms + r.scale_ms + r.add_ms - r.wall_ms) <= 1e-6 * r.wall_ms
    assert r.device_ms >= r.wall_ms * 0.99
    plan = pe.DevicePlan(g, 3, "real", 0, 1)
    plan.upload(pr.stat, 1)
    for _ in range(2):
        rep = plan.execute(1)
        assert rep.conv_ms > 0 and rep.add_ms > 0 and rep.device_ms >= rep.wall_ms * 0.99


def test_sharded_report_times_the_exchange_on_the_device():
    """a sharded plan's finish report: conv stage, exchange (conv end ->
    addition-stage start), additions, all from the device's own clock"""
    pr = pe.gen_benchmark("p1", 15, 2, seed=7)
    g = pe.build_jobgraph_shape(pr.n, pr.d, pr.nvars, pr.indices)
    plans = [pe.DevicePlan(g, 2, "real", 0, 1, rank=r, nranks=2) for r in range(2)]
    plans[0].set_peer(1, plans[1])
    plans[1].set_peer(0, plans[0])
    for p in plans:
        p.upload(pr.stat, 1)
        p.execute(1)
    for p in plans:
        p.gather_peers(1)
    for p in plans:
        fin = p.finish(1)
        assert fin.conv_ms > 0 and fin.add_ms > 0 and fin.exchange_ms >= 0
        assert abs(fin.conv_ms + fin.exchange_ms + fin.scale_ms + fin.add_ms - fin.wall_ms) <= 1e-6 * fin.wall_ms + 1e-6


@pytest.mark.parametrize("m", [1, 2])
def test_sharded_plan_with_an_empty_rank(m):
    """more ranks than independent job groups (one monomial, 3 ranks): the
    ranks without conv jobs still run the exchange and the exact addition
    tree, and every rank's result equals one device's (m=1: the CTA-local
    layer walk with groups that have no jobs on a rank)"""
    pe_g = pe.GraphArrays  # noqa: F841 (import check)
    rng = np.random.default_rng(11)
    p = md_instance(rng, m, False, nmax=3, Nmax=1, dmin=5, dmax=5)
    g = pe.build_jobgraph_shape(p.n, p.d, p.nvars, p.idx)
    st = p.stat.reshape(p.P * p.m, *p.stat.shape[2:])
    want, _, _ = pe.DevicePlan(g, m, "real", 0, 1).run(st, 1)
    plans = [pe.DevicePlan(g, m, "real", 0, 1, rank=r, nranks=3) for r in range(3)]
    for p1 in plans:
        for p2 in plans:
            if p2 is not p1:
                p1.set_peer(p2.rank, p2)
        p1.upload(st, 1)
        rep = p1.execute(1)
        assert rep.conv_ms >= 0
    for p1 in plans:
        p1.gather_peers(1)
    for p1 in plans:
        fin = p1.finish(1)
        assert fin.add_ms >= 0 and fin.wall_ms >= 0
        vg, _ = p1.download(1)
        assert_bitwise(vg, want, f"rank {p1.rank}/3 of a one-monomial polynomial")
