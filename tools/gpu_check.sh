#!/bin/bash
# one gpurun call: GPU parity suite + C2 bench (+ optional extra workloads)
# usage: tools/gpu_check.sh [workload ...]
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for w in c2 "$@"; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));print('$w', round(d['ms_per_step'],3),'ms', round(d['value'],2), d['unit'], 'frac', d.get('roofline',{}).get('frac'), 'e2e', d['e2e']['value'], 'clk', d['clocks'])" || tail -5 gpurun_out/bench_$w.err
done
