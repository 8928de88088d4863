for v in default fpref; do
  if [ $v = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
  for m in 2 3 4; do python tools/variant_time.py --workload c3 --m $m; done
  python tools/diag/shape_time.py p1:31:2 p2:40:3
done
