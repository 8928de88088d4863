timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ctl" -x > gpurun_out/r2b_pytest_ctl.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_ctl.log | tail -5
python tools/diag/layers.py --workload c3 --m 1
for v in default ctlu8 ctlr4u4 ctlr2u4; do
  if [ $v = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
  python tools/variant_time.py --workload c3 --m 1
done
