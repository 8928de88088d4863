for v in default fm6 fm8; do
  if [ $v = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
  python tools/variant_time.py --workload c3 --m 2
  python tools/variant_time.py --workload c1
done
