timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b_pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2b_pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python tools/variant_time.py --workload c3 --m 1
timeout 900 python bench.py --workload c3 --m 1 > gpurun_out/r2b_bench_c3_m1.json 2> gpurun_out/r2b_bench_c3_m1.err; python -c "import json;d=json.load(open('gpurun_out/r2b_bench_c3_m1.json'));r=d['roofline'];print('c3_m1', round(d['ms_per_eval'],3),'ms/eval', round(d['value'],2), r['conv_path'], 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],2), 'clk', d['clocks']['sm_mhz'], d['clocks']['samples'], d['clocks']['reasons'])"
