#!/bin/bash
mkdir -p gpurun_out
B=paper_2101_10881_b200/pseval_b200
timeout 600 $B bench p2 --degree 152 --precision 1 2 3 4 5 8 10 --csv gpurun_out/p2sweep_auto.csv > gpurun_out/p2sweep_auto.log 2>&1
PSE_CONV_MODE=layer timeout 600 $B bench p2 --degree 152 --precision 1 2 3 4 5 8 10 --csv gpurun_out/p2sweep_layer.csv > gpurun_out/p2sweep_layer.log 2>&1
cat gpurun_out/p2sweep_auto.csv gpurun_out/p2sweep_layer.csv
for wv in 8 16 32 64 128; do
  timeout 600 python bench.py --workload c5 --points 128 --wave $wv --steps 2 --warmup 1 --no-cpu > gpurun_out/c5_w$wv.json 2>gpurun_out/c5_w$wv.err
  python -c "import json;d=json.load(open('gpurun_out/c5_w$wv.json'));print('c5 wave $wv', round(d['ms_per_step'],2), d['value'], d['roofline']['frac'])" || tail -3 gpurun_out/c5_w$wv.err
done
PSE_CONV_MODE=flow timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/flow_c2_full python tools/profile_run.py --workload c2 > gpurun_out/prof_flow.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_conv_flow -c 1 -o gpurun_out/flow_c3h_full python tools/profile_run.py --workload c3h >> gpurun_out/prof_flow.log 2>&1
tail -2 gpurun_out/prof_flow.log
