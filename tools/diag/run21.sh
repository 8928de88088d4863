timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ctl or cta or full_size" > gpurun_out/r2b_pytest_ctl.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_ctl.log | tail -5
python tools/diag/layers.py --workload c3 --m 1
python tools/variant_time.py --workload c3 --m 1
python tools/variant_time.py --workload c3h --m 1
timeout 600 python bench.py --workload c3 --m 1 > gpurun_out/r2b_bench_c3_m1.json 2> gpurun_out/r2b_bench_c3_m1.err; python -c "import json;d=json.load(open('gpurun_out/r2b_bench_c3_m1.json'));r=d['roofline'];print(round(d['ms_per_eval'],3),'ms/eval', round(d['value'],2), r['conv_path'], 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],2), 'clk', d['clocks']['sm_mhz'], d['clocks']['samples'], d['clocks']['reasons'])"
ncu --set full --import-source on --clock-control none -k k_conv_ctl -c 1 -o gpurun_out/r2b_ctl_c3_m1 -f python tools/profile_run.py --workload c3 --m 1 > /dev/null 2>&1; echo "ctl rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_traffic_c3_m1.csv python tools/profile_run.py --workload c3 --m 1 > /dev/null 2>&1; echo "traffic m1 rc=$?"
