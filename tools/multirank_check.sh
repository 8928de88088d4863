#!/bin/bash
# the bench's multi-rank paths with two ranks sharing the one GPU of a gpurun
# box (gloo for the host-side barriers / reductions): `bench.py --gpus 2`
# relaunches itself under torch.distributed.run. Plumbing checks, not scaling
# numbers (both ranks time-share one device).
export PSE_DIST_BACKEND=gloo
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_shard2.json 2> gpurun_out/bench_shard2.err; echo "monomials (default) rc=$?"; tail -c 600 gpurun_out/bench_shard2.json
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --shard points --points 4 --no-cpu > gpurun_out/bench_points2.json 2> gpurun_out/bench_points2.err; echo "points rc=$?"; tail -c 400 gpurun_out/bench_points2.json
PSE_EXCHANGE=collective timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --workload c1 > gpurun_out/bench_shard2_coll.json 2> gpurun_out/bench_shard2_coll.err; echo "monomials collective c1 rc=$?"; tail -c 400 gpurun_out/bench_shard2_coll.json
timeout 900 python bench.py --impl reference --gpus 2 --steps 1 --warmup 3 --workload c1 > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref2.json
