"""Host logic of the banded conv paths (no GPU): the task schedule that the
wave and dataflow kernels run. pse_band_schedule_stats builds the same
schedule a plan builds and raises if any warp descriptor would wait on a
later one (the dataflow kernel's no-deadlock condition), so these tests
check completeness (every band x segment task scheduled exactly once, in a
slot of the right width) and that condition on the benchmark graphs and on
random shapes."""
import numpy as np
import pytest

import paper_2101_10881_b200 as pe
from paper_2101_10881_b200.pseval import band_schedule_stats

from instances import int_instance


def expected_tasks(g, W):
    nb = 1 + g.d // W
    copies = g.copy_job_count()
    return (g.conv_job_count() - copies) * nb * (nb + 1) // 2 + copies * nb


def slots_per_job(d, W):
    """occupied 8-lane slots of one non-copy job: rectangular tasks W/8,
    diagonal tasks W/16"""
    nb = 1 + d // W
    return nb * (nb - 1) // 2 * (W // 8) + nb * (W // 16)


def shape(pid, d):
    p = pe.gen_benchmark("p2" if pid == "p2h" else pid, d, 1, seed=7, with_static=False)
    nv, ix = np.asarray(p.nvars), np.asarray(p.indices)
    if pid == "p2h":  # even cyclic windows, as bench.py's C3'
        starts = np.concatenate([[0], np.cumsum(nv)])
        keep = np.arange(0, len(nv), 2)
        ix = np.concatenate([ix[starts[k]:starts[k + 1]] for k in keep])
        nv = nv[keep]
    return pe.build_jobgraph_shape(p.n, d, nv, ix)


@pytest.mark.parametrize("pid", ["p1", "p2h", "p3"])
@pytest.mark.parametrize("W", [16, 32])
@pytest.mark.parametrize("flow", [True, False])
def test_benchmark_graphs_schedule_every_task_once(pid, W, flow):
    d = 152
    g = shape(pid, d)
    st = band_schedule_stats(g, W, flow)
    assert st["jobs"] == g.conv_job_count()
    assert st["tasks"] == expected_tasks(g, W)
    assert g.copy_job_count() == 0
    assert st["slots"] == g.conv_job_count() * slots_per_job(d, W)
    assert st["descriptors"] * 4 >= st["slots"]
    # slots are packed densely: at most a few percent of descriptor slots empty
    assert st["slots"] >= 0.95 * 4 * st["descriptors"]
    if flow:
        assert st["waves"] == 1
    else:
        # every wave waits for the previous one: at least the dependency depth
        assert st["waves"] >= g.conv_layer_sizes().__len__() + (1 + d // W) - 1
    assert st["makespan_steps"] > 0


def test_narrow_bands_shorten_the_critical_path_of_deep_graphs():
    """C3' (64-layer chains): the makespan estimate that picks the band width
    prefers 16-wide bands; C2 (4 layers, 1820 monomials) is work-bound."""
    deep, wide = shape("p2h", 152), shape("p1", 152)
    assert band_schedule_stats(deep, 16)["makespan_steps"] < band_schedule_stats(deep, 32)["makespan_steps"]
    w16, w32 = band_schedule_stats(wide, 16), band_schedule_stats(wide, 32)
    assert abs(w16["makespan_steps"] - w32["makespan_steps"]) < 0.1 * w32["makespan_steps"]


def test_random_graphs_with_copies_and_in_place_folds():
    """random shapes (monomials of one variable give copy jobs, n_k >= 3 the
    in-place coefficient fold) at degrees across band boundaries"""
    rng = np.random.default_rng(77)
    for it in range(60):
        p = int_instance(rng, False, nmax=7, Nmax=9, dmax=1)
        d = int(rng.choice([0, 1, 8, 15, 16, 17, 31, 32, 33, 47, 64, 100, 152]))
        g = pe.build_jobgraph_shape(p.n, d, p.nvars, p.idx)
        for W in (16, 32):
            for flow in (True, False):
                st = band_schedule_stats(g, W, flow, procs=int(rng.integers(1, 300)))
                assert st["tasks"] == expected_tasks(g, W), (it, d, W, flow)


def test_rejects_bad_band_width():
    g = shape("p1", 8)
    with pytest.raises(pe.InvalidArgument):
        band_schedule_stats(g, 24)
