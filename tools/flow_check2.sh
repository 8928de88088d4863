#!/bin/bash
mkdir -p gpurun_out
B=paper_2101_10881_b200/pseval_b200
timeout 300 $B bench p2 --degree 152 --precision 1 2 3 4 5 8 10 --csv gpurun_out/p2sweep_auto.csv > /dev/null 2>&1; echo -n "auto p2: "; cut -d, -f3,11 gpurun_out/p2sweep_auto.csv | tr '\n' ' '; echo
for w in c3h c2; do python tools/profile_run.py --workload $w --reps 3; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "flow" 2>&1 | tail -1
