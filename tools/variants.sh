#!/bin/bash
# A/B timing of tuning builds: tools/variants.sh "<variant> ..." "<workload> ..."
mkdir -p gpurun_out
for w in $2; do
  for v in $1; do
    if [ "$v" = default ]; then unset PSE_LIB_VARIANT; else export PSE_LIB_VARIANT=$v; fi
    timeout 300 python tools/variant_time.py --workload $w 2>&1 | tail -1
  done
done | tee -a gpurun_out/variants.log
