#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "flow or band" > gpurun_out/pytest_band.log 2>&1; echo "pytest flow rc=$?"; tail -1 gpurun_out/pytest_band.log
B=paper_2101_10881_b200/pseval_b200
timeout 300 $B bench p2 --degree 152 --precision 1 2 3 4 5 8 10 --csv gpurun_out/p2sweep_auto.csv > /dev/null 2>&1; echo -n "auto p2: "; cut -d, -f3,11 gpurun_out/p2sweep_auto.csv | tr '\n' ' '; echo
for W in 16 32; do PSE_BAND_W=$W timeout 300 $B bench p2 --degree 152 --precision 3 5 8 --csv gpurun_out/p2sweep_w$W.csv > /dev/null 2>&1; echo -n "W=$W p2: "; cut -d, -f3,11 gpurun_out/p2sweep_w$W.csv | tail -3 | tr '\n' ' '; echo; done
for w in c3h c2 c1; do python tools/profile_run.py --workload $w --reps 3; done
