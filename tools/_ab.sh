# A/B: tuning builds (libpse_b200_<v>.so) vs the working tree, conv-stage times + checksum
# usage: tools/_ab.sh "<variants>" "<workload:m> ..."
mkdir -p gpurun_out
for spec in $2; do
  w=${spec%%:*}; m=${spec##*:}
  for v in $1; do
    if [ $v = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
    timeout 300 python tools/variant_time.py --workload $w --m $m --reps 5 2>&1 | tail -1
  done
done
