#!/bin/bash
for w in c2 c4; do python tools/profile_run.py --workload $w --reps 3; PSE_CONV_MODE=flow python tools/profile_run.py --workload $w --reps 3; PSE_CONV_MODE=flow PSE_BAND_W=16 python tools/profile_run.py --workload $w --reps 3; done
