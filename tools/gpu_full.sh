#!/bin/bash
# full round check: GPU parity suite, smoke, bench lines for every config, reference arm
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for w in c2 c1 c3 c3h c4; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$w.json'));r=d['roofline'];print('$w', round(d['ms_per_step'],3),'ms', round(d['value'],2), d['unit'], r['conv_path'], 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['ms_per_call'],3), 'cpu', d.get('cpu_baseline',{}).get('ms_per_eval'))" || tail -5 gpurun_out/bench_$w.err
done
timeout 1200 python bench.py --workload c5 --points 256 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python -c "import json;d=json.load(open('gpurun_out/bench_c5.json'));print('c5', round(d['ms_per_eval'],3),'ms/pt', round(d['value'],2), d['roofline']['conv_path'], 'frac', round(d['roofline']['frac'],3))" || tail -5 gpurun_out/bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
