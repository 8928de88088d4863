for v in default aeo edv; do
  if [ $v = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
  python tools/variant_time.py --workload c2
  python tools/variant_time.py --workload c3h
done
