#!/bin/bash
# round-2 measurement pass on one gpurun box: GPU parity suite, smoke, bench
# lines for every BASELINE configuration (+ the C3 precision sweep, C5 on 256
# points) and the reference arm; outputs under gpurun_out/r2_*
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() {  # name, bench args...
  local n=$1; shift
  timeout 1200 python bench.py "$@" > gpurun_out/r2_bench_$n.json 2> gpurun_out/r2_bench_$n.err
  python -c "import json;d=json.load(open('gpurun_out/r2_bench_$n.json'));r=d['roofline'];print('$n', round(d['ms_per_eval'],3),'ms/eval', round(d['value'],2), d['unit'], r['conv_path'], 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],2), 'clk', d['clocks']['sm_mhz'], d['clocks']['samples'], d['clocks']['reasons'], 'cpu', (d.get('cpu_baseline') or {}).get('ms_per_eval'))" || tail -5 gpurun_out/r2_bench_$n.err
}
run c2 --workload c2 --steps 20 --warmup 5
run c1 --workload c1
run c3 --workload c3
run c3h --workload c3h
run c4 --workload c4
for m in 1 2 3 4 5 8; do run c3_m$m --workload c3 --m $m; done
run c5_256 --workload c5 --points 256 --steps 3 --warmup 3 --no-cpu
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err; tail -c 400 gpurun_out/r2_bench_ref.json
