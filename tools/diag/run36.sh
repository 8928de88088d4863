python tools/variant_time.py --workload c3h
PSE_BAND_W=32 python tools/variant_time.py --workload c3h
PSE_FLOW_SLACK=0.5 python tools/variant_time.py --workload c3h
PSE_FLOW_SLACK=2 python tools/variant_time.py --workload c3h
PSE_FLOW_PROCS=0.8 python tools/variant_time.py --workload c3h
PSE_FLOW_PROCS=1.25 python tools/variant_time.py --workload c3h
PSE_BAND_W=16 python tools/variant_time.py --workload c3
PSE_FLOW_SLACK=0.5 python tools/variant_time.py --workload c3
