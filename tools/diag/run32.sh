for w in c3 c3h c4; do
  python tools/variant_time.py --workload $w
  PSE_CONV_MODE=layer python tools/variant_time.py --workload $w
  PSE_CONV_MODE=flow python tools/variant_time.py --workload $w
done
for m in 3 5 8; do
  python tools/variant_time.py --workload c2 --m $m
  PSE_CONV_MODE=layer python tools/variant_time.py --workload c2 --m $m
  PSE_CONV_MODE=flow python tools/variant_time.py --workload c2 --m $m
done
