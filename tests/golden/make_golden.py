"""Generate the golden fixtures in tests/golden/ from the REFERENCE engine
itself (oracle/_ref/libpseval_ref.so, compiled from /root/reference/proj/src
by oracle/Makefile). Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

The fixtures travel with the repo so the C restatement (oracle/) and the CUDA
engine can be pinned on machines without /root/reference.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))

import pyoracle as po  # noqa: E402
from instances import int_instance, md_instance  # noqa: E402

LEVELS = [1, 2, 3, 4, 5, 8, 10]


def save_problem(name, p: po.Problem, **arrays):
    np.savez_compressed(os.path.join(HERE, name), n=p.n, d=p.d, m=p.m, cplx=int(p.cplx), nvars=p.nvars, idx=p.idx,
                        exps=p.exps if p.exps is not None else np.zeros(0, np.int32), stat=p.stat, **arrays)


def main():
    assert po.has_ref(), "build oracle/_ref first (make -C oracle)"
    meta = {"source": "oracle/_ref/libpseval_ref.so (reference engine compiled from /root/reference/proj/src)"}

    # md ops: random_md pairs + edge values, every precision level
    for m in LEVELS:
        x = po.random_md(31 * m, m, 1500, lib="ref")
        y = po.random_md(37 * m, m, 1500, lib="ref")
        edge = np.zeros((6, m))
        edge[1, 0] = 1.0
        edge[2, 0] = -1.0
        edge[3] = -0.0
        edge[4] = x[0]
        edge[5] = -x[1]
        X = np.concatenate([x, np.repeat(edge, 6, 0)])
        Y = np.concatenate([y, np.tile(edge, (6, 1))])
        np.savez_compressed(os.path.join(HERE, f"md_m{m}.npz"), x=X, y=Y,
                            add=po.md_op("add", X, Y, "ref"), sub=po.md_op("sub", X, Y, "ref"),
                            mul=po.md_op("mul", X, Y, "ref"))

    # known answers: RNG stream, cost tables, graph shapes, FLOP totals
    meta["rng_u64_seed7"] = [int(v) for v in po.rng_u64(7, 8, "ref")]
    meta["mix_seed_7_1<<32"] = po.mix_seed(7, 1 << 32, "ref")
    meta["costs"] = {str(m): po.cost(m, "ref") for m in LEVELS}
    meta["graphs"] = {}
    for pid in ("p1", "p2", "p3"):
        p = po.ref_gen_benchmark(pid, 2, 1)
        g = po.graph(p, "ref")
        conv_sizes = np.bincount(g["conv"][:, 0])[1:].tolist()
        add_sizes = np.bincount(g["add"][:, 0])[1:].tolist()
        meta["graphs"][pid] = dict(total_slots=g["total_slots"], conv=len(g["conv"]), add=len(g["add"]),
                                   conv_layers=conv_sizes, add_layers=add_sizes, copies=g["ncopy"],
                                   conv_sha=int(np.bitwise_xor.reduce((g["conv"] * np.arange(1, len(g["conv"]) + 1)[:, None]).ravel())),
                                   add_sha=int(np.bitwise_xor.reduce((g["add"] * np.arange(1, len(g["add"]) + 1)[:, None]).ravel())))
    p1 = po.ref_gen_benchmark("p1", 2, 1)
    meta["flops_p1_d152_deca"] = [po.flop_count(p1, 397, 3089, w, "ref", d=152) for w in (0, 1, 2)]

    # whole-engine outputs (value + gradients), reference run_sequential
    for pid, d, m in [("p1", 15, 2), ("p1", 8, 1), ("p1", 8, 4), ("p1", 31, 2), ("p2", 3, 3), ("p3", 3, 5),
                      ("p1", 6, 10), ("p1", 5, 8)]:
        p = po.ref_gen_benchmark(pid, d, m, seed=7)
        vg = po.evaluate(p, "ref")
        np.save(os.path.join(HERE, f"vg_{pid}_d{d}_m{m}.npy"), vg)
    # C1 with complex mode (same shapes, seed 7)
    p = po.ref_gen_benchmark("p1", 6, 2, cplx=True, seed=7)
    np.save(os.path.join(HERE, "vg_p1_d6_m2_cplx.npy"), po.evaluate(p, "ref"))

    # random instances: integer (bitwise vs eval_direct) and full precision
    rng = np.random.default_rng(2101)
    for i in range(12):
        p = int_instance(rng, i % 2 == 1)
        save_problem(f"int_{i:02d}.npz", p, vg=po.evaluate(p, "ref"), direct=po.eval_direct(p, "ref"))
    for i, m in enumerate([2, 3, 4, 5, 8, 10]):
        p = md_instance(rng, m, cplx=i % 2 == 1, with_exponents=True)
        save_problem(f"md_{m}.npz", p, vg=po.evaluate(p, "ref"))

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote", len(os.listdir(HERE)), "files")


if __name__ == "__main__":
    main()
