#!/bin/bash
mkdir -p gpurun_out
for m in 1 2 3 4 5 8; do
  timeout 600 python bench.py --workload c3 --m $m > gpurun_out/bench_c3_m$m.json 2> gpurun_out/bench_c3_m$m.err
  python -c "import json;d=json.load(open('gpurun_out/bench_c3_m$m.json'));r=d['roofline'];print('m=$m', round(d['ms_per_step'],3),'ms', round(d['value'],2), r['conv_path'], 'frac', round(r['frac'],3), 'cpu', d.get('cpu_baseline',{}).get('ms_per_eval'))" || tail -3 gpurun_out/bench_c3_m$m.err
done
B=paper_2101_10881_b200/pseval_b200
timeout 300 $B bench p2 --degree 152 --precision 1 2 3 4 5 8 10 --csv gpurun_out/p2sweep_auto.csv > /dev/null 2>&1; cut -d, -f3,11 gpurun_out/p2sweep_auto.csv | tr '\n' ' '
