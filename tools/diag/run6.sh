python tools/diag/layers.py --workload c3 --m 1
python tools/diag/layers.py --workload c3h --m 1
PSE_CONV_MODE=cta python tools/diag/layers.py --workload c3 --m 1
