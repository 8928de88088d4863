python tools/diag/layers.py --workload c3 --m 1
PSE_CTL_DBG=1 python tools/diag/layers.py --workload c3 --m 1
PSE_CTL_DBG=2 python tools/diag/layers.py --workload c3 --m 1
PSE_CTL_DBG=3 python tools/diag/layers.py --workload c3 --m 1
