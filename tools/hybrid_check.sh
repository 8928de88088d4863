#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for w in c2 c4 c3h; do python tools/profile_run.py --workload $w --reps 3; PSE_CONV_MODE=layer python tools/profile_run.py --workload $w --reps 3; done
for g in 2 8; do PSE_CONV_GROUPS=$g python tools/profile_run.py --workload c2 --reps 3; done
