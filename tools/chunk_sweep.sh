#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "flow" > gpurun_out/pytest_band.log 2>&1; echo "pytest flow rc=$?"; tail -1 gpurun_out/pytest_band.log
B=paper_2101_10881_b200/pseval_b200
for c in 1 4 16 64; do
  echo -n "chunk $c: "; PSE_FLOW_CHUNK=$c timeout 300 $B bench p2 --degree 152 --precision 1 2 5 10 --csv gpurun_out/chunk_$c.csv > /dev/null 2>&1; cut -d, -f3,11 gpurun_out/chunk_$c.csv | tail -4 | tr '\n' ' '; echo
done
for c in 1 4 16; do PSE_FLOW_CHUNK=$c PSE_CONV_MODE=flow python tools/profile_run.py --workload c2 --reps 2; done
