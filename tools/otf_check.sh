#!/bin/bash
for w in c2 c4; do
  echo -n "old: "; PSE_LIB_VARIANT=old python tools/profile_run.py --workload $w --reps 3
  echo -n "otf minb4: "; PSE_CONV_MINB=4 python tools/profile_run.py --workload $w --reps 3
  echo -n "otf minb5: "; PSE_CONV_MINB=5 python tools/profile_run.py --workload $w --reps 3
done
echo -n "old: "; PSE_LIB_VARIANT=old python tools/profile_run.py --workload c3h --reps 3
echo -n "otf: "; python tools/profile_run.py --workload c3h --reps 3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "md_ops or conv or c1 or p1 or md_instances" 2>&1 | tail -1
