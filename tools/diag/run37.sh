timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ctl or empty_rank or sharding or batched or c1_" -x > gpurun_out/r2b_pytest_sub.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed|Error" gpurun_out/r2b_pytest_sub.log | tail -5
timeout 120 python tools/diag/layers.py --workload c3 --m 1
for v in default t1; do
  if [ $v = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
  for w in c3 c3h c2 c4 c1; do timeout 120 python tools/variant_time.py --workload $w --m 1; done
done
