#!/bin/bash
# round-2 (second half) measurement pass on one gpurun box: GPU parity suite,
# smoke, bench lines for every BASELINE configuration, the C3 precision sweep,
# C5, the reference arm, complex timings; outputs under gpurun_out/r2b_*
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2b_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() {  # name, bench args...
  local n=$1; shift
  timeout 1500 python bench.py "$@" > gpurun_out/r2b_bench_$n.json 2> gpurun_out/r2b_bench_$n.err
  python -c "import json;d=json.load(open('gpurun_out/r2b_bench_$n.json'));r=d['roofline'];print('$n', round(d['ms_per_eval'],3),'ms/eval', round(d['value'],2), d['unit'], r['conv_path'], 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],2), 'clk', d['clocks']['sm_mhz'], d['clocks']['samples'], d['clocks']['reasons'], 'cpu', (d.get('cpu_baseline') or {}).get('ms_per_eval'))" || tail -5 gpurun_out/r2b_bench_$n.err
}
run c2_driver --gpus 1 --steps 20 --warmup 5
run c1 --workload c1
run c3 --workload c3
run c3h --workload c3h
run c4 --workload c4
for m in 1 2 3 4 5 8; do run c3_m$m --workload c3 --m $m; done
run c5_256 --workload c5 --points 256 --steps 3 --warmup 3 --no-cpu
run c5_1024 --workload c5 --steps 1 --warmup 3 --no-cpu
timeout 600 python tools/cplx_time.py > gpurun_out/r2b_cplx_time.txt 2>&1; cat gpurun_out/r2b_cplx_time.txt
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2b_bench_ref_driver.json 2> gpurun_out/r2b_bench_ref_driver.err; tail -c 300 gpurun_out/r2b_bench_ref_driver.json
