timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ctl" -x > gpurun_out/r2b_pytest_ctl.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_ctl.log | tail -5
python tools/diag/layers.py --workload c3 --m 1
python tools/variant_time.py --workload c3 --m 1
PSE_LIB_VARIANT=ctlblk python tools/variant_time.py --workload c3 --m 1
python tools/variant_time.py --workload c3h --m 1
python tools/variant_time.py --workload c2 --m 1
