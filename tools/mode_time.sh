#!/bin/bash
# conv-stage time of workloads x precisions x conv paths (PSE_CONV_MODE):
#   tools/mode_time.sh "<workload ...>" "<m ...>" "<mode ...>"   (mode "auto" = the planner's pick)
mkdir -p gpurun_out
for w in $1; do for m in $2; do for mode in $3; do
  if [ "$mode" = auto ]; then unset PSE_CONV_MODE; else export PSE_CONV_MODE=$mode; fi
  echo -n "$mode "; timeout 300 python tools/variant_time.py --workload $w --m $m 2>&1 | tail -1
done; done; done | tee -a gpurun_out/mode_time.log
