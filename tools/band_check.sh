#!/bin/bash
# banded / dataflow conv path: parity + timing sweep against the layered path
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "flow or band" > gpurun_out/pytest_band.log 2>&1; echo "pytest flow rc=$?"; tail -3 gpurun_out/pytest_band.log
rm -f gpurun_out/sweep.log
for w in c3h c3 c2 c4; do
  bash tools/sweep.sh "PSE_CONV_MODE=layer:$w:3" "PSE_CONV_MODE=flow PSE_FLOW_SLACK=0.15:$w:3" "PSE_CONV_MODE=flow PSE_FLOW_SLACK=0.4:$w:3"
done
cat gpurun_out/sweep.log
