#!/bin/bash
# re-entry check of round 2: GPU parity suite, smoke, C2 bench, small-precision and complex timings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2b_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() {  # name, bench args...
  local n=$1; shift
  timeout 1200 python bench.py "$@" > gpurun_out/r2b_bench_$n.json 2> gpurun_out/r2b_bench_$n.err
  python -c "import json;d=json.load(open('gpurun_out/r2b_bench_$n.json'));r=d['roofline'];print('$n', round(d['ms_per_eval'],3),'ms/eval', round(d['value'],2), d['unit'], r['conv_path'], 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],2), 'clk', d['clocks']['sm_mhz'], d['clocks']['samples'], d['clocks']['reasons'])" || tail -5 gpurun_out/r2b_bench_$n.err
}
run c2 --workload c2 --no-cpu
run c3h --workload c3h --no-cpu
run c4 --workload c4 --no-cpu
for m in 1 2 3 4 5; do run c3_m$m --workload c3 --m $m --no-cpu; done
timeout 600 python tools/cplx_time.py 2>&1 | tail -5
