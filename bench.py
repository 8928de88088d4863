#!/usr/bin/env python
"""Benchmark: evaluation + full gradient of a polynomial at a power series
truncated at degree d in multiple-double precision (arXiv 2101.10881), on the
B200 engine, in the reference's metric (BASELINE.json).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--impl ours|reference]

A step = one evaluation + full gradient of the workload (C1-C4: one
polynomial at one point; C5: every point of the batch). With --gpus N > 1 the
script re-launches itself under torch.distributed.run (one rank per GPU);
one polynomial is then sharded by monomials (strong scaling, exact addition
tree after a peer-memory gather) and the C5 batch by points
(no data-path collective). Step time = CUDA events / the kernels' own
%globaltimer stamps on each rank's device, max over ranks.

Printed (rank 0): ONE JSON line. `value` = model TFLOPS (the reference's
flop_count with reporting_cost, executor.cpp:233-252 / multidouble.cpp:70-75,
divided by device time with inputs resident in HBM); `e2e` = the same metric
through the public C-ABI call pse_plan_run with pinned host buffers (H2D of
the static region + D2H of value and gradients inside the timed region);
`roofline` = the conv stage (the dominant kernels) of the same timed launches
in algorithmic binary64 ops per second against the FP64 issue rate measured
live on this GPU; `cpu_baseline` = the reference's own engine (run_bench,
bench.cpp:17-50) on this host's cores.

--impl reference: the reference's own CPU engine (oracle/_ref, compiled from
the reference sources) on the same workload, config and metric; that process
never loads this package's native library.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TFLOPS & ms per eval+gradient at d=152 deca double (1 GPU; 2/4/8 if sharded)"

WORKLOADS = {
    # name: (polynomial id, d, m, points, description)
    "c1": ("p1", 15, 2, 1, "C1: p1 (16 vars, 1820 monomials of 4 vars), d=15, double-double"),
    "c2": ("p1", 152, 10, 1, "C2: p1 (16 vars, 1820 monomials of 4 vars), d=152, deca double"),
    "c3": ("p2", 152, 10, 1, "C3: p2 (128 vars, 128 cyclic monomials of 64 vars), d=152"),
    "c3h": ("p2h", 152, 10, 1, "C3': p2h (128 vars, 64 monomials of 64 vars), d=152, deca double"),
    "c4": ("p3", 152, 10, 1, "C4: p3 (128 vars, 8128 products of two variables), d=152, deca double"),
    "c5": ("p2h", 152, 10, 1024, "C5: 1024 points x p2h, d=152, deca double, sharded over GPUs"),
}
L2_NOTE = "256 MiB buffer rewritten between timed steps (arena also > L2)"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def shard_mode(args, wl):
    if args.shard:
        return args.shard
    return "points" if wl == "c5" else "monomials"


def config_for(args, wl, world):
    """The workload description both arms print (identical dicts)."""
    pid, d, m, points, desc = WORKLOADS[wl]
    if args.points:
        points = args.points
    sh = shard_mode(args, wl)
    par = "1 GPU" if world == 1 else (f"points x{world} (no data-path collective)" if sh == "points" else
                                      f"monomials x{world} (exact addition tree after a peer-memory gather)")
    return {"workload": desc, "id": pid, "d": d, "m": m, "points": points, "parallelism": par, "l2": L2_NOTE}


def cpu_info():
    """threads this process may use, physical cores, SMT (for the CPU legs)"""
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    try:
        import psutil

        phys = psutil.cpu_count(logical=False) or threads
    except Exception:
        phys = threads
    logical = os.cpu_count() or threads
    return threads, {"physical_cores": phys, "logical_cpus": logical,
                     "smt": f"{max(1, logical // max(1, phys))} threads per core"}


# ----------------------------------------------------------------- problems
def make_static(pid: str, d: int, m: int, points: range):
    """Packed shape + static block [Q][len(points)][top][d+1] from the
    product's generator (bit-identical to gen.cpp:50-71). Point b takes the
    coefficients of seed 7 and the inputs z of seed 1000+b (SURVEY.md 8(d)
    C5); a single C1-C4 point is exactly gen_benchmark(id, d, m, real, 7)."""
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


def ref_problem(pid: str, d: int, m: int, point: int = 0):
    """The same problem built by the REFERENCE library's own gen_benchmark
    (oracle/_ref): no code of this package is loaded."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    base_id = "p2" if pid == "p2h" else pid
    p = po.ref_gen_benchmark(base_id, d, m, seed=7)
    if point:
        zb = po.ref_gen_benchmark(base_id, d, m, seed=1000 + point)
        p.stat[:, :, 1 + p.N:] = zb.stat[:, :, 1 + p.N:]
    if pid == "p2h":
        keep = np.arange(0, p.N, 2)
        starts = np.concatenate([[0], np.cumsum(p.nvars)])
        idx = np.concatenate([p.idx[starts[k]:starts[k + 1]] for k in keep]).astype(np.int32)
        stat = np.concatenate([p.stat[:, :, :1], p.stat[:, :, 1 + keep], p.stat[:, :, 1 + p.N:]], axis=2)
        p = po.Problem(p.n, p.d, p.m, False, p.nvars[keep].copy(), idx, None, np.ascontiguousarray(stat), "p2h")
    return po, p


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock, clock-event (throttle) reasons and power sampled every few
    ms through NVML in a thread while the timed steps run; entering returns
    after the first sample, so even short timed regions are covered."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, device: int, interval_s: float = 0.005):
        self.device, self.interval = device, interval_s
        self.rows, self.max_mhz, self.src = [], None, None
        self._stop = threading.Event()
        self._thread = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self._nvml_index(nv))
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            first = threading.Event()

            def run():
                while not self._stop.is_set():
                    try:
                        sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                        try:
                            pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                        except Exception:
                            pw = None
                        self.rows.append((sm, rs, pw))
                    except Exception:
                        pass
                    first.set()
                    time.sleep(self.interval)

            self._thread = threading.Thread(target=run, daemon=True)
            self._thread.start()
            first.wait(2.0)
            self.src = "nvml"
        except Exception:
            self.src = None
        return self

    def _nvml_index(self, nv):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.device < len(ids) and ids[self.device].isdigit():
                return int(ids[self.device])
        return self.device

    def __exit__(self, *a):
        self._stop.set()
        if self._thread:
            self._thread.join(1.0)

    def summary(self):
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"], "samples": 0}
        reasons = sorted({k for _, rs, _ in rows for k, bit in self.REASONS.items() if rs & bit})
        pw = [p for _, _, p in rows if isinstance(p, (int, float))]
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(pw, default=None), "source": self.src}


# ----------------------------------------------------------------- CPU legs
def reference_time(po, p, threads: int, min_ms: float = 0.0):
    """The reference's own run_bench (bench.cpp:17-50: build the graph, fold,
    stage, run_parallel on `threads` workers) on the WHOLE graph of one
    point; repeats (median) until about min_ms of CPU time. Returns (ms per
    eval+gradient, repeats)."""
    _, _, wall, _ = po.ref_run_bench(p, threads, 1)
    reps = 1
    if wall < min_ms:
        reps = int(min(9, max(1, min_ms // max(wall, 1e-3))))
        _, _, wall, _ = po.ref_run_bench(p, threads, reps)
    return wall, reps


def reference_arm(args, wl):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref = the reference sources compiled unmodified) on this host's
    cores, same metric / config; rank 0 only. Inputs and the FLOP count come
    from the reference library too, so this process never maps the
    product's libpse_b200.so."""
    rank, _, world = env_rank()
    if rank != 0:
        return
    pid, d, m, points, desc = WORKLOADS[wl]
    threads, cinfo = cpu_info()
    po, p = ref_problem(pid, d, m, point=0)
    if not po.has_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return
    _, _, rep_add, rep_mul = po.cost(m, "ref")
    model_ops = po.flop_count(p, rep_add, rep_mul, lib="ref")
    times = []
    for s in range(args.warmup + args.steps):
        ms, _ = reference_time(po, p, threads)
        if s >= args.warmup:
            times.append(ms)
    ms = statistics.median(times)
    value = model_ops / (ms * 1e-3) / 1e12
    total = sum(times)
    sample = (f"reference run_bench (bench.cpp:17-50) = run_parallel({threads} threads) over the whole graph of one "
              f"point, {args.steps} timed runs (median)" + (f"; a step is one of the {points} points" if points > 1 else ""))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "ms_per_eval": ms,
        "higher_is_better": True, "scaling": "strong" if shard_mode(args, wl) == "monomials" else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (gen_benchmark seed 7; reference library)",
        "config": config_for(args, wl, world),
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": threads, "kind": "reference", "sample": sample,
                         **cinfo, "timed_s": round(total / 1e3, 2)},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "model_double_ops_per_eval": model_ops,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(pid, d, m, model_ops):
    """our arm's cpu_baseline: the same reference run_bench on one point,
    whole graph (bounded: ~10-15 s at m=10 on 16 threads)."""
    threads, cinfo = cpu_info()
    po, p = ref_problem(pid, d, m)
    if not po.has_ref():
        return None
    ms, reps = reference_time(po, p, threads, min_ms=2000.0)
    return {"value": model_ops / (ms * 1e-3) / 1e12, "unit": "TFLOPS", "cores": threads, "kind": "reference",
            "sample": f"reference run_bench (bench.cpp:17-50), run_parallel({threads} threads), whole graph of one "
                      f"point, median of {reps}", "ms_per_eval": ms, **cinfo}


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
    "cta": "k_conv_cta<{m},real> (one block per independent job group and point, CTA-local dataflow)",
    "cta_layers": "k_conv_ctl<{m},real> (one block per independent job group and point, its layers in order)",
}


def repeat_count(t_eval_ms: float, red_dev=None) -> int:
    """Evaluations per timed step: short evaluations repeat so that a step
    lasts >= 25 ms and the clock sampler sees it (C1, small precisions). The
    count is the max over ranks -- every rank must run the same number of
    evaluations, since a sharded evaluation has collectives."""
    from paper_2101_10881_b200 import dist as D

    mine = max(1, int(np.ceil(25.0 / max(t_eval_ms, 1e-3))))
    return int(D.max_over_ranks(float(mine), red_dev))


def gpu_setup(args):
    import torch

    from paper_2101_10881_b200 import dist as D

    rank, local, world = env_rank()
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    # NCCL for the barriers / max-over-ranks reductions; PSE_DIST_BACKEND=gloo
    # lets several ranks share one GPU when testing the multi-rank paths
    backend = os.environ.get("PSE_DIST_BACKEND", "nccl")
    red_dev = torch.device(f"cuda:{dev}") if backend == "nccl" else None
    if world > 1:
        D.init(backend)
    return rank, world, dev, red_dev, D


def roofline_block(m, path, conv_ops_total, conv_ms_total, peak, clk, sms, wl, extra=None):
    achieved = conv_ops_total / (conv_ms_total * 1e-3) if conv_ms_total > 0 else 0.0
    peak_ops = max(peak["dadd"], peak["dfma"])
    out = {
        "bound": "fp64", "kernel": CONV_KERNEL[path].format(m=m), "conv_path": path,
        "achieved": achieved / 1e12, "peak": peak_ops / 1e12, "unit": "Tops/s (binary64, algorithmic)",
        "frac": achieved / peak_ops, "traffic": load_traffic(wl, path),
        "traffic_unit": "DRAM bytes of the conv stage per evaluation point (ncu, profiles/ncu_traffic.json)",
        "peak_source": "measured live: pse_fp64_peak (independent DADD/DFMA chains on every SM, best of two shapes)",
        "peak_nominal": sms * 64 * (clk.get("sm_max_mhz") or 0) * 1e6 / 1e12,
        "peak_nominal_note": "SMs x 64 FP64 lanes x max SM clock (binary64 instructions/s)",
        "timing": "conv stage of the timed launches themselves: the kernels' %globaltimer stamps (first conv "
                  "block start -> last conv job end)",
    }
    if extra:
        out.update(extra)
    return out


def ours_points(args, wl):
    """Each rank evaluates its own contiguous range of points (C5; C1-C4 with
    --shard points): no data-path collective."""
    import torch

    import paper_2101_10881_b200 as pe

    rank, world, dev, red_dev, D = gpu_setup(args)
    cfg = config_for(args, wl, world)
    pid, d, m, total_points = cfg["id"], cfg["d"], cfg["m"], cfg["points"]
    b0, b1 = D.point_range(total_points, rank, world)
    mine = range(b0, b1)
    n, N, nvars, idx, stat = make_static(pid, d, m, mine)
    g = pe.build_jobgraph_shape(n, d, nvars, idx)
    wave = max(1, min(len(mine), args.wave))
    plan = pe.DevicePlan(g, m, "real", dev, wave)
    Q = stat.shape[0]
    waves = [range(s, min(s + wave, len(mine))) for s in range(0, len(mine), wave)]
    model_ops = pe.flop_count(g, d, "real", pe.reporting_cost(m))
    conv_ops = conv_alg_ops(g, d, m)
    peak = pe.fp64_peak(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    # every point's static inputs resident in HBM before timing starts; a
    # multi-wave batch stages each wave from there (D2D) inside the step
    stat_dev = torch.from_numpy(np.ascontiguousarray(stat)).to(f"cuda:{dev}")
    torch.cuda.synchronize(dev)
    pstream = torch.cuda.ExternalStream(plan.stream(), device=f"cuda:{dev}")
    single = len(waves) == 1

    def upload(w):
        plan.upload_ptr(stat_dev.data_ptr(), len(w), total=len(mine), first=w.start)

    if single:
        upload(waves[0])

    def evaluate_once():
        """(device ms, conv-stage ms, kernel launches) of one pass over this
        rank's points"""
        if single:
            r = plan.execute(len(waves[0]))
            return r.device_ms, r.conv_ms, r.kernel_launches
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        conv = 0.0
        launches = 0
        e0.record(pstream)
        for w in waves:
            upload(w)
            r = plan.execute(len(w))
            conv += r.conv_ms
            launches += r.kernel_launches + 1
        e1.record(pstream)
        e1.synchronize()
        return e0.elapsed_time(e1), conv, launches

    for _ in range(args.warmup):
        t_eval = evaluate_once()[0]
    # short evaluations repeat inside a step so that every step lasts >= 25 ms
    # and the clock sampler sees the timed region (C1, small precisions); the
    # same count on every rank
    reps = repeat_count(t_eval, red_dev)
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    walls, convs, launches = [], [], 0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.random_(0, 255)
            torch.cuda.synchronize(dev)
            w = c = 0.0
            for _ in range(reps):
                a, b, l = evaluate_once()
                w, c, launches = w + a, c + b, launches + l
            walls.append(w)
            convs.append(c)
    clocks = clk.summary()
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    total_ms = D.max_over_ranks(sum(walls), red_dev)
    conv_ms = sum(convs)
    evals = args.steps * reps
    value = model_ops * total_points * evals / (total_ms * 1e-3) / 1e12
    path = plan.conv_path(wave)

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
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "ms_per_eval": total_ms / evals / len(mine),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_benchmark seed 7 coefficients; inputs seed 7 or 1000+point)",
        "config": cfg, "evals_per_step": reps, "layout": {"points_per_gpu": len(mine), "wave": wave},
        "model_double_ops_per_eval": model_ops, "conv_alg_ops_per_eval": conv_ops,
        "roofline": roofline_block(m, path, conv_ops * len(mine) * evals, conv_ms, peak, clocks, sms, wl,
                                   {"conv_ms_per_eval": conv_ms / (len(mine) * evals), "alg_ops_per_eval": conv_ops}),
        "e2e": {"value": e2e_value, "unit": "TFLOPS", "ms_per_call": e2e_total / args.steps,
                "h2d_bytes_per_step": int(Q * nb * pw * 8), "d2h_bytes_per_step": int(Q * nb * (n + 1) * (d + 1) * 8)},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_leg(pid, d, m, model_ops)
    print(json.dumps(line), flush=True)


def ours_monomials(args, wl):
    """ONE polynomial (seed 7) over the ranks: each GPU runs the conv jobs of
    its share of the monomials, the addition-stage term slots are gathered
    from the peers' arenas (CUDA IPC: NVLink peer memory) and every rank runs
    the exact addition tree -- bit-identical to one GPU. At N=1 this is the
    plain single-GPU evaluation."""
    import torch

    import paper_2101_10881_b200 as pe

    rank, world, dev, red_dev, D = gpu_setup(args)
    cfg = config_for(args, wl, world)
    pid, d, m = cfg["id"], cfg["d"], cfg["m"]
    n, N, nvars, idx, stat = make_static(pid, d, m, range(1))
    g = pe.build_jobgraph_shape(n, d, nvars, idx)
    plan = pe.DevicePlan(g, m, "real", dev, 1, rank=rank, nranks=world)
    p2p = world > 1 and os.environ.get("PSE_EXCHANGE", "p2p") == "p2p" and D.connect_peers(plan)
    model_ops = pe.flop_count(g, d, "real", pe.reporting_cost(m))
    conv_ops = conv_alg_ops(g, d, m)
    peak = pe.fp64_peak(dev)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    Q = stat.shape[0]
    stat1 = np.ascontiguousarray(stat[:, 0])
    plan.upload(stat1, 1)

    def evaluate_once():
        """(device ms of the whole evaluation, conv ms, exchange ms, launches);
        sharded: conv start -> last addition layer by the kernels' stamps on
        this device (the exchange and barriers included)"""
        if world == 1:
            r = plan.execute(1)
            return r.device_ms, r.conv_ms, 0.0, r.kernel_launches
        rep, fin = D.evaluate_sharded(plan, 1, p2p=p2p)
        return fin.wall_ms, fin.conv_ms, fin.exchange_ms, rep.kernel_launches + fin.kernel_launches + (1 if p2p else 0)

    for _ in range(args.warmup):
        t_eval = evaluate_once()[0]
    # the same repeat count on every rank: each evaluation has collectives
    reps = repeat_count(t_eval, red_dev)
    if world > 1:
        torch.distributed.barrier()
    walls, convs, exs, launches = [], [], [], 0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            flush.random_(0, 255)
            torch.cuda.synchronize(dev)
            w = c = x = 0.0
            for _ in range(reps):
                a, b, e, l = evaluate_once()
                w, c, x, launches = w + a, c + b, x + e, launches + l
            walls.append(w)
            convs.append(c)
            exs.append(x)
    clocks = clk.summary()
    total = D.max_over_ranks(sum(walls), red_dev)
    conv_max = D.max_over_ranks(sum(convs), red_dev)
    evals = args.steps * reps
    path = plan.conv_path(1)

    # ---- e2e: pinned host inputs -> (sharded) evaluation -> value/gradients on the host
    import ctypes as C

    from paper_2101_10881_b200._lib import lib

    pw = stat.shape[2] * (d + 1)
    hin = lib().pse_host_alloc(Q * pw * 8)
    hout = lib().pse_host_alloc(Q * (n + 1) * (d + 1) * 8)
    pin_in = np.ctypeslib.as_array(C.cast(hin, C.POINTER(C.c_double)), (Q, stat.shape[2], d + 1))
    pin_out = np.ctypeslib.as_array(C.cast(hout, C.POINTER(C.c_double)), (Q, 1, n + 1, d + 1))
    pin_in[...] = stat1
    pstream = torch.cuda.ExternalStream(plan.stream(), device=f"cuda:{dev}")
    e2es = []
    for s in range(args.warmup + args.steps):
        flush.random_(0, 255)
        torch.cuda.synchronize(dev)
        if world == 1:
            _, _, rep = plan.run(pin_in, 1, out=pin_out)
            ms = rep.e2e_ms
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(pstream)
            plan.upload(pin_in, 1)
            D.evaluate_sharded(plan, 1, p2p=p2p)
            plan.download(1, out=pin_out)
            e1.record(pstream)
            e1.synchronize()
            ms = e0.elapsed_time(e1)
        if s >= args.warmup:
            e2es.append(ms)
    e2e_total = D.max_over_ranks(sum(e2es), red_dev)
    lib().pse_host_free(hin)
    lib().pse_host_free(hout)
    if rank != 0:
        return
    ms = total / evals
    extra = {"conv_ms_per_eval": conv_max / evals, "alg_ops_per_eval": conv_ops}
    if world > 1:
        extra.update({"note": "conv ops of all ranks over the slowest rank's conv stage",
                      "exchange_ms_per_eval_rank0": sum(exs) / evals})
    line = {
        "metric": METRIC, "value": model_ops / (ms * 1e-3) / 1e12, "unit": "TFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps, "ms_per_eval": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_benchmark seed 7)", "config": cfg, "evals_per_step": reps,
        "model_double_ops_per_eval": model_ops, "conv_alg_ops_per_eval": conv_ops,
        "roofline": roofline_block(m, path, conv_ops * evals, conv_max, peak, clocks, sms, wl, extra),
        "e2e": {"value": model_ops / (e2e_total / args.steps * 1e-3) / 1e12, "unit": "TFLOPS",
                "ms_per_call": e2e_total / args.steps,
                "h2d_bytes_per_step": int(Q * pw * 8) * world, "d2h_bytes_per_step": int(Q * (n + 1) * (d + 1) * 8) * world},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_leg(pid, d, m, model_ops)
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks (one per
    GPU) of this same command on this node."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--wave", type=int, default=128, help="points per device launch (C5)")
    ap.add_argument("--shard", default="", choices=["", "points", "monomials"],
                    help="N>1: monomials = one polynomial split over the ranks (strong scaling, exact; default for "
                         "C1-C4); points = each rank evaluates its own points (weak scaling; default for C5)")
    ap.add_argument("--points", type=int, default=0,
                    help="override the workload's point count (total, sharded by points)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--m", type=int, default=0, choices=[0, 1, 2, 3, 4, 5, 8, 10],
                    help="override the precision level (C3's sweep: 1/2/3/4/5/8/10)")
    args = ap.parse_args()
    if args.m:
        pid, d, m, pts, desc = WORKLOADS[args.workload]
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
        WORKLOADS[args.workload] = (pid, d, args.m, pts, desc)
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit("--gpus must be at least 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        reference_arm(args, args.workload)
    elif shard_mode(args, args.workload) == "monomials":
        ours_monomials(args, args.workload)
    else:
        ours_points(args, args.workload)


if __name__ == "__main__":
    main()
