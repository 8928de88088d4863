for w in c2 c4 c1; do
  python tools/variant_time.py --workload $w --m 1
  PSE_CONV_MODE=ctl python tools/variant_time.py --workload $w --m 1
done
