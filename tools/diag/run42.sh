for v in default m2t512 m2t1024; do
  if [ $v = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
  python tools/variant_time.py --workload c3 --m 2
  PSE_CONV_MODE=cta python tools/variant_time.py --workload c3 --m 2
done
for m in 3 4; do
  python tools/variant_time.py --workload c3 --m $m
  PSE_CONV_MODE=cta python tools/variant_time.py --workload c3 --m $m
done
