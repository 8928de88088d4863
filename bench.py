#!/usr/bin/env python
"""Benchmark: evaluation + full gradient of a polynomial at a power series
truncated at degree d in multiple-double precision (arXiv 2101.10881), on the
B200 engine, in the reference's metric (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

A step = one evaluation + full gradient of every point a rank owns (one
point per GPU for C1-C4; the C5 batch is sharded across ranks). Multi-GPU runs
are launched by torchrun, one rank per GPU; points shard with no data-path
collective (weak scaling), timing is the max over ranks.

Printed (rank 0): ONE JSON line. `value` = model TFLOPS (the reference's
flop_count with reporting_cost, executor.cpp:233-252 / multidouble.cpp:70-75,
divided by device time with inputs resident in HBM); `e2e` = the same metric
through the public C-ABI call pse_plan_run with pinned host buffers (H2D of
the static region + D2H of value and gradients inside the timed region);
`roofline` = the dominant kernel (the conv layers) in algorithmic binary64
ops per second against the FP64 issue rate measured live on this GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TFLOPS & ms per eval+gradient at d=152 deca double (1 GPU; 2/4/8 if sharded)"

WORKLOADS = {
    # name: (polynomial id, d, m, points per GPU, description)
    "c1": ("p1", 15, 2, 1, "C1: p1 (16 vars, 1820 monomials of 4 vars), d=15, double-double"),
    "c2": ("p1", 152, 10, 1, "C2: p1 (16 vars, 1820 monomials of 4 vars), d=152, deca double"),
    "c3": ("p2", 152, 10, 1, "C3: p2 (128 vars, 128 cyclic monomials of 64 vars), d=152"),
    "c3h": ("p2h", 152, 10, 1, "C3': p2h (128 vars, 64 monomials of 64 vars), d=152, deca double"),
    "c4": ("p3", 152, 10, 1, "C4: p3 (128 vars, 8128 products of two variables), d=152, deca double"),
    "c5": ("p2h", 152, 10, 1024, "C5: 1024 points x p2h, d=152, deca double, sharded over GPUs"),
}


# ----------------------------------------------------------------- problems
def make_static(pid: str, d: int, m: int, points: range):
    """Packed shape + static block [Q][len(points)][top][d+1]. Point b takes
    the coefficients of seed 7 and the inputs z of seed 1000+b (SURVEY.md
    8(d) C5); a single C1-C4 point is exactly gen_benchmark(id, d, m, real, 7)."""
    import paper_2101_10881_b200 as pe

    base_id = "p2" if pid == "p2h" else pid
    base = pe.gen_benchmark(base_id, d, m, seed=7)
    nvars, idx, st = base.nvars, base.indices, base.stat
    n, N = base.n, base.N
    if pid == "p2h":  # the literal "64 monomials of 64 vars": p2's even windows
        keep = np.arange(0, 128, 2)
        starts = np.concatenate([[0], np.cumsum(nvars)])
        idx = np.concatenate([idx[starts[k]:starts[k + 1]] for k in keep]).astype(np.int32)
        nvars = nvars[keep].copy()
        st = np.concatenate([st[:, :1], st[:, 1 + keep], st[:, 1 + N:]], axis=1)
        N = len(keep)
    Q = st.shape[0]
    top = 1 + N + n
    out = np.empty((Q, len(points), top, d + 1), np.float64)
    for j, b in enumerate(points):
        out[:, j] = st
        if not (len(points) == 1 and b == 0):
            zb = pe.gen_benchmark(base_id, d, m, seed=1000 + b).stat
            out[:, j, 1 + N:] = zb[:, 1 + base.N:]
    return n, N, nvars, idx, out


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 8 and f[0].replace(".", "").isdigit():
                    rows.append(f)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[7]) for r in rows if r[7] not in ("", "[N/A]"))}


# ----------------------------------------------------------------- CPU leg
def cpu_sample(pid, d, m, threads: int, target_jobs: int):
    """Reference CPU engine (oracle/_ref = the reference's own sources, else
    the C port) on a bounded sample: the first J conv jobs of conv layer 1
    (static, full-precision inputs: every conv job of the graph costs the
    same) plus ALL addition layers. Returns (ms per eval+gradient
    extrapolated to the whole graph, kind, cores, sample description)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    import paper_2101_10881_b200 as pe

    n, N, nvars, idx, st = make_static(pid, d, m, range(1))
    prob = po.Problem(n, d, m, False, nvars, idx, None, st[:, 0].reshape(1, m, -1, d + 1))
    g = pe.build_jobgraph_shape(n, d, nvars, idx)
    C = g.conv_job_count() - g.copy_job_count()
    if po.has_ref():
        conv_ms, add_ms, wall_ms, J = po.ref_bench_sample(prob, threads, target_jobs)
        total = conv_ms * C / J + add_ms
        if total < 2000.0:  # cheap enough (C1): the reference's own run_bench on the whole graph
            _, _, wall, _ = po.ref_run_bench(prob, threads, 3)
            return wall, "reference", threads, (f"reference run_bench (bench.cpp:17-50), run_parallel({threads} "
                                                f"threads), whole graph: {C} conv + {g.add_job_count()} add jobs, "
                                                f"median of 3")
        return total, "reference", threads, (f"reference run_parallel({threads} threads): first {J} of {C} conv "
                                             f"jobs of layer 1 timed and scaled x{C / J:.1f}, plus all {g.add_job_count()} add jobs")
    J = max(1, min(8, target_jobs))
    ms, J = po.port_time_conv_jobs(prob, J)
    return ms * C / J, "port", 1, f"C port, 1 thread: {J} conv jobs of layer 1 scaled x{C / J:.1f} (adds omitted)"


def reference_arm(args, wl):
    """--impl reference: the reference's own CPU implementation of the path
    on this host's cores, same metric/config, rank 0 only."""
    rank, _, world = (int(os.environ.get(k, v)) for k, v in (("RANK", 0), ("LOCAL_RANK", 0), ("WORLD_SIZE", 1)))
    if rank != 0:
        return
    import paper_2101_10881_b200 as pe

    pid, d, m, ppg, desc = WORKLOADS[wl]
    threads = os.cpu_count() or 1
    n, N, nvars, idx, _ = make_static(pid, d, m, range(1))
    g = pe.build_jobgraph_shape(n, d, nvars, idx)
    model_ops = pe.flop_count(g, d, "real", pe.reporting_cost(m))
    jobs = min(g.conv_layer_sizes()[0], max(64, threads * 24))
    times = []
    kind = cores = sample = None
    for s in range(args.warmup + args.steps):
        ms, kind, cores, sample = cpu_sample(pid, d, m, threads, jobs)
        if s >= args.warmup:
            times.append(ms)
    ms = statistics.median(times)
    points = 1
    value = model_ops / (ms * 1e-3) / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_eval": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_benchmark seed 7)", "config": {"workload": desc, "points": points},
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU leg
def conv_alg_ops(g, d: int, m: int) -> int:
    import paper_2101_10881_b200 as pe

    c = pe.instrumented_cost(m)
    C = g.conv_job_count() - g.copy_job_count()
    return C * ((d + 1) * (d + 2) // 2 * c.mul_cost + d * (d + 1) // 2 * c.add_cost)


def load_traffic(wl: str, path: str):
    """DRAM bytes of the conv stage per evaluation point for this workload and
    conv path, from the committed ncu captures (profiles/ncu_traffic.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))[f"{wl}/{path}"]["dram_bytes_per_eval"]
    except Exception:
        return None


CONV_KERNEL = {
    "layered": "k_conv<{m},real> (one launch per conv layer and monomial group; split prod/accum for small layers)",
    "waves": "k_conv_band<{m},real> (one launch per scheduled wave of band x segment tasks)",
    "dataflow": "k_conv_flow<{m},real> (one persistent launch per evaluation wave)",
    "hybrid": "k_conv<{m},real> for the large conv layers, then k_conv_flow<{m},real> for the trailing small ones",
}


def ours(args, wl):
    import torch

    import paper_2101_10881_b200 as pe
    from paper_2101_10881_b200 import dist as D

    rank, local, world = D.env_rank()
    dev = local % max(1, torch.cuda.device_count())
    # NCCL for the barrier / max-over-ranks timing reduction; PSE_DIST_BACKEND
    # =gloo lets several ranks share one GPU when testing the multi-rank path
    backend = os.environ.get("PSE_DIST_BACKEND", "nccl")
    red_dev = torch.device(f"cuda:{dev}") if backend == "nccl" else None
    if world > 1:
        torch.cuda.set_device(dev)
        D.init(backend)
    pid, d, m, ppg, desc = WORKLOADS[wl]
    if args.points:
        ppg = args.points
    total_points = ppg * world if wl != "c5" else ppg
    b0, b1 = D.point_range(total_points, rank, world)
    mine = range(b0, b1)
    n, N, nvars, idx, stat = make_static(pid, d, m, mine)
    g = pe.build_jobgraph_shape(n, d, nvars, idx)
    wave = min(len(mine), args.wave)
    plan = pe.DevicePlan(g, m, "real", dev, max(1, wave))
    Q = stat.shape[0]
    waves = [range(s, min(s + wave, len(mine))) for s in range(0, len(mine), wave)]
    model_ops = pe.flop_count(g, d, "real", pe.reporting_cost(m))
    conv_ops = conv_alg_ops(g, d, m)
    peak = pe.fp64_peak(dev)
    sms_count = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_ops = max(peak["dadd"], peak["dfma"])

    # L2 flush buffer (> 126 MB L2), written between timed steps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")

    # every point's static inputs resident in HBM before timing starts; a
    # multi-wave batch stages each wave from there (D2D) inside the step
    stat_dev = torch.from_numpy(np.ascontiguousarray(stat)).to(f"cuda:{dev}")
    pstream = torch.cuda.ExternalStream(plan.stream(), device=f"cuda:{dev}")

    def upload(w):
        plan.upload_ptr(stat_dev.data_ptr(), len(w), total=len(mine), first=w.start)

    stats = {}
    single_wave = len(waves) == 1
    if single_wave:
        upload(waves[0])

    def step(detail=False):
        """one evaluation of every point this rank owns; device time from CUDA
        events on the engine's stream around the whole step (the evaluation
        is one CUDA-graph launch per wave); with detail, the phases run
        un-captured with events between them, for the conv share"""
        conv = 0.0
        launches = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(pstream)
        for w in waves:
            if not single_wave:
                upload(w)
                launches += 1
            r = plan.execute(len(w), detail=detail)
            stats["alg"] = r.alg_op_count
            conv += r.conv_ms
            launches += r.kernel_launches
        e1.record(pstream)
        e1.synchronize()
        return e0.elapsed_time(e1), conv, launches

    for _ in range(args.warmup):
        step()
        step(detail=True)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    walls, convs, launches = [], [], 0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.random_(0, 255)
            torch.cuda.synchronize(dev)
            w, c, l = step()
            walls.append(w)
            convs.append(c)
            launches += l
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    my_total = sum(walls)
    total_ms = D.max_over_ranks(my_total, red_dev)
    ms_per_step = total_ms / args.steps
    value = model_ops * total_points * args.steps / (total_ms * 1e-3) / 1e12
    # conv share of the step (roofline): the same steps with per-phase events
    convs = []
    for _ in range(args.steps):
        flush.random_(0, 255)
        torch.cuda.synchronize(dev)
        convs.append(step(detail=True)[1])
    conv_ms = sum(convs)
    path = plan.conv_path(wave)
    achieved = conv_ops * len(mine) * args.steps / (conv_ms * 1e-3)

    # ---- e2e: public C-ABI call with pinned host buffers, one wave per call
    import ctypes as C

    from paper_2101_10881_b200._lib import lib

    w0 = waves[0]
    nb = len(w0)
    pw = stat.shape[2] * (d + 1)
    hin = lib().pse_host_alloc(Q * nb * pw * 8)
    hout = lib().pse_host_alloc(Q * nb * (n + 1) * (d + 1) * 8)
    pin_in = np.ctypeslib.as_array(C.cast(hin, C.POINTER(C.c_double)), (Q, nb, stat.shape[2], d + 1))
    pin_out = np.ctypeslib.as_array(C.cast(hout, C.POINTER(C.c_double)), (Q, nb, n + 1, d + 1))
    pin_in[...] = stat[:, w0.start:w0.stop]
    e2e_ms = []
    for s in range(args.warmup + args.steps):
        flush.random_(0, 255)
        torch.cuda.synchronize(dev)
        _, _, rep = plan.run(pin_in, nb, out=pin_out)
        if s >= args.warmup:
            e2e_ms.append(rep.e2e_ms)
    e2e_total = D.max_over_ranks(sum(e2e_ms), red_dev)
    e2e_points = nb * D.sum_over_ranks(1.0, red_dev)
    e2e_value = model_ops * e2e_points * args.steps / (e2e_total * 1e-3) / 1e12
    lib().pse_host_free(hin)
    lib().pse_host_free(hout)

    if rank != 0:
        return
    alg_ops = stats["alg"]
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "ms_per_eval": ms_per_step * world / total_points,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_benchmark seed 7 coefficients; inputs seed 7 or 1000+point)",
        "config": {"workload": desc, "id": pid, "d": d, "m": m, "points": total_points,
                   "points_per_gpu": len(mine), "wave": wave, "parallelism": f"points x{world}" if world > 1 else "1 GPU",
                   "l2": "256 MiB buffer rewritten between timed steps (arena also > L2)"},
        "model_double_ops_per_eval": model_ops,
        "alg_ops_per_eval": alg_ops,
        "conv_alg_ops_per_eval": conv_ops,
        "roofline": {
            "bound": "fp64", "kernel": CONV_KERNEL[path].format(m=m), "conv_path": path,
            "achieved": achieved / 1e12, "peak": peak_ops / 1e12, "unit": "Tops/s (binary64, algorithmic)",
            "frac": achieved / peak_ops, "traffic": load_traffic(wl, path),
            "traffic_unit": "DRAM bytes of the conv stage per evaluation point (ncu, profiles/ncu_traffic.json)",
            "peak_source": "measured live: pse_fp64_peak (independent DADD/DFMA chains on every SM, best of two shapes)",
            "peak_nominal": sms_count * 64 * (clk.summary().get("sm_max_mhz") or 0) * 1e6 / 1e12,
            "peak_nominal_note": "SMs x 64 FP64 lanes x max SM clock (binary64 instructions/s)",
            "conv_ms_per_eval": conv_ms / (len(mine) * args.steps),
            "alg_ops_per_eval": conv_ops,
        },
        "e2e": {"value": e2e_value, "unit": "TFLOPS", "ms_per_call": e2e_total / args.steps,
                "h2d_bytes_per_step": int(Q * nb * pw * 8), "d2h_bytes_per_step": int(Q * nb * (n + 1) * (d + 1) * 8)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        jobs = min(g.conv_layer_sizes()[0], max(64, threads * 24))
        cms, kind, cores, sample = cpu_sample(pid, d, m, threads, jobs)
        line["cpu_baseline"] = {"value": model_ops / (cms * 1e-3) / 1e12, "unit": "TFLOPS", "cores": cores,
                                "kind": kind, "sample": sample, "ms_per_eval": cms}
    print(json.dumps(line), flush=True)


def ours_sharded(args, wl):
    """--shard monomials: ONE polynomial (C2/C4 point, seed 7) strong-scaled
    over the ranks -- each GPU runs the conv jobs of its share of the
    monomials, the addition-stage term slots are all-gathered over NCCL
    (NVLink), and every rank runs the exact addition tree (bit-identical to
    one GPU). Step time = conv (events) + exchange (host clock around
    pack/all-gather/unpack, synchronised) + addition stage (events), max over
    ranks."""
    import time

    import torch

    import paper_2101_10881_b200 as pe
    from paper_2101_10881_b200 import dist as D

    rank, local, world = D.env_rank()
    dev = local % max(1, torch.cuda.device_count())
    backend = os.environ.get("PSE_DIST_BACKEND", "nccl")
    red_dev = torch.device(f"cuda:{dev}") if backend == "nccl" else None
    torch.cuda.set_device(dev)
    if world > 1:
        D.init(backend)
    pid, d, m, _, desc = WORKLOADS[wl]
    n, N, nvars, idx, stat = make_static(pid, d, m, range(1))
    g = pe.build_jobgraph_shape(n, d, nvars, idx)
    plan = pe.DevicePlan(g, m, "real", dev, 1, rank=rank, nranks=world)
    # exchange: peer gather over mapped arenas (CUDA IPC: NVLink peer memory)
    # unless PSE_EXCHANGE=collective or IPC is unavailable
    p2p = world > 1 and os.environ.get("PSE_EXCHANGE", "p2p") == "p2p" and D.connect_peers(plan)
    model_ops = pe.flop_count(g, d, "real", pe.reporting_cost(m))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    pinned = torch.from_numpy(np.ascontiguousarray(stat)).pin_memory()

    def step(e2e: bool):
        t0 = time.perf_counter()
        if e2e:
            plan.upload_ptr(pinned.data_ptr(), 1)
        if world > 1:
            conv, ex, fin = D.evaluate_sharded(plan, 1, p2p=p2p)
        else:
            r = plan.execute(1, detail=True)
            conv, ex, fin = r.conv_ms, 0.0, r.wall_ms - r.conv_ms
        if e2e and rank == 0:
            plan.download(1)
        return conv + ex + fin, conv, (time.perf_counter() - t0) * 1e3

    plan.upload(stat, 1)
    for _ in range(args.warmup):
        step(False)
    if world > 1:
        torch.distributed.barrier()
    walls, convs, e2es = [], [], []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.random_(0, 255)
            torch.cuda.synchronize(dev)
            w, c, _ = step(False)
            walls.append(w)
            convs.append(c)
    for _ in range(args.steps):
        e2es.append(step(True)[2])
    total = D.max_over_ranks(sum(walls), red_dev)
    e2e_total = D.max_over_ranks(sum(e2es), red_dev)
    if rank != 0:
        return
    ms = total / args.steps
    line = {
        "metric": METRIC, "value": model_ops / (ms * 1e-3) / 1e12, "unit": "TFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_eval": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_benchmark seed 7)",
        "config": {"workload": desc + " -- one polynomial sharded by monomials", "id": pid, "d": d, "m": m,
                   "points": 1, "parallelism": f"monomials x{world} (exact addition tree after "
                                               f"{'a peer-memory gather' if p2p else 'an all-gather'})",
                   "l2": "256 MiB buffer rewritten between timed steps"},
        "conv_ms_rank0": sum(convs) / args.steps,
        "e2e": {"value": model_ops / (e2e_total / args.steps * 1e-3) / 1e12, "unit": "TFLOPS",
                "ms_per_call": e2e_total / args.steps, "timing": "host clock, synchronised",
                "h2d_bytes_per_step": int(stat.nbytes), "d2h_bytes_per_step": int(plan.Q * (n + 1) * (d + 1) * 8)},
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--wave", type=int, default=128, help="points per device launch (C5)")
    ap.add_argument("--shard", default="points", choices=["points", "monomials"],
                    help="points: each rank evaluates its own points (weak scaling, default); monomials: one "
                         "polynomial split over the ranks (strong scaling, exact)")
    ap.add_argument("--points", type=int, default=0,
                    help="override the workload's point count (per GPU for C1-C4, total for C5)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--m", type=int, default=0, choices=[0, 1, 2, 3, 4, 5, 8, 10],
                    help="override the precision level (C3's sweep: 1/2/3/4/5/8/10)")
    args = ap.parse_args()
    if args.m:
        pid, d, m, ppg, desc = WORKLOADS[args.workload]
        if args.m != m:
            names = {1: "double", 2: "double-double", 3: "triple double", 4: "quad double", 5: "penta double",
                     8: "octo double", 10: "deca double"}
            for old in sorted(names.values(), key=len, reverse=True):  # "double-double" before "double"
                if desc.endswith(", " + old):
                    desc = desc[: -len(old)] + names[args.m]
                    break
            else:
                desc += ", " + names[args.m]
            desc += f" (m={args.m})"
        WORKLOADS[args.workload] = (pid, d, args.m, ppg, desc)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args, args.workload)
    elif args.shard == "monomials":
        ours_sharded(args, args.workload)
    else:
        ours(args, args.workload)


if __name__ == "__main__":
    main()
