#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "flow" > gpurun_out/pytest_band.log 2>&1; echo "pytest flow rc=$?"; tail -1 gpurun_out/pytest_band.log
B=paper_2101_10881_b200/pseval_b200
for W in 0 32 64; do
  echo -n "W=$W p2: "; PSE_BAND_W=$W timeout 300 $B bench p2 --degree 152 --precision 1 2 3 4 5 8 10 --csv gpurun_out/sw.csv > /dev/null 2>&1; cut -d, -f3,11 gpurun_out/sw.csv | tail -7 | tr '\n' ' '; echo
done
for W in 0 64; do echo -n "W=$W "; PSE_BAND_W=$W python tools/profile_run.py --workload c3h --reps 3; done
python tools/profile_run.py --workload c2 --reps 3
