python tools/variant_time.py --workload c1
PSE_CONV_MODE=ctl python tools/variant_time.py --workload c1
PSE_CONV_MODE=cta python tools/variant_time.py --workload c1
PSE_CONV_MODE=layer python tools/variant_time.py --workload c1
