for v in default sk100 sk400 sk1600; do
  if [ $v = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
  python tools/variant_time.py --workload c4
  python tools/variant_time.py --workload c2
done
