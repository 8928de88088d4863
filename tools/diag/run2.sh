mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b_pytest_full.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_full.log | tail -30
run() {  # name, bench args...
  local n=$1; shift
  timeout 1200 python bench.py "$@" > gpurun_out/r2b_bench_$n.json 2> gpurun_out/r2b_bench_$n.err
  python -c "import json;d=json.load(open('gpurun_out/r2b_bench_$n.json'));r=d['roofline'];print('$n', round(d['ms_per_eval'],3),'ms/eval', round(d['value'],2), d['unit'], r['conv_path'], 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],2), 'clk', d['clocks']['sm_mhz'], d['clocks']['samples'], d['clocks']['reasons'])" || tail -5 gpurun_out/r2b_bench_$n.err
}
run c2 --workload c2 --no-cpu
