#!/bin/bash
B=paper_2101_10881_b200/pseval_b200
timeout 300 $B bench p2 --degree 152 --precision 1 2 3 4 10 --csv gpurun_out/sw.csv > /dev/null 2>&1; cut -d, -f3,11 gpurun_out/sw.csv | tr '\n' ' '; echo
python tools/profile_run.py --workload c3h --reps 3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "flow" 2>&1 | tail -1
