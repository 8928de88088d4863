#!/bin/bash
# two ranks sharing the one GPU of a gpurun box (gloo for the host-side collectives)
export PSE_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo "points rc=$?"; tail -c 400 gpurun_out/bench_2rank.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 3 --warmup 3 --shard monomials > gpurun_out/bench_shard2.json 2> gpurun_out/bench_shard2.err; echo "monomials rc=$?"; tail -c 400 gpurun_out/bench_shard2.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_ref2.json 2> gpurun_out/bench_ref2.err; echo "ref rc=$?"; tail -c 200 gpurun_out/bench_ref2.json
