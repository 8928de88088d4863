# conv time of C2 / C4 by the number of concurrent monomial groups (PSE_CONV_GROUPS)
for g in 1 2 4 8 16; do
  PSE_CONV_GROUPS=$g python tools/variant_time.py --workload c2 | sed "s/^/groups=$g /"
  PSE_CONV_GROUPS=$g python tools/variant_time.py --workload c4 | sed "s/^/groups=$g /"
done
