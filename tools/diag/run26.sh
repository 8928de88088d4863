for m in 2 3 4; do
  python tools/variant_time.py --workload c3 --m $m
  PSE_BAND_W=16 python tools/variant_time.py --workload c3 --m $m
  PSE_BAND_W=32 python tools/variant_time.py --workload c3 --m $m
  PSE_FLOW_SLACK=0.5 python tools/variant_time.py --workload c3 --m $m
  PSE_FLOW_SLACK=2 python tools/variant_time.py --workload c3 --m $m
done
