timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "md_ or identities or edge or c1_ or full_size or integer or instances" -x > gpurun_out/r2b_pytest_sub.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_sub.log | tail -5
for v in default tord0; do
  if [ $v = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
  python tools/variant_time.py --workload c2
  python tools/variant_time.py --workload c4
  python tools/variant_time.py --workload c3h
  python tools/variant_time.py --workload c3 --m 3
done
