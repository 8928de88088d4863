timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -k "sharding or empty_rank or ctl or cta or c1_ or p1_bitwise or p2_p3 or integer" > gpurun_out/r2b_pytest_sub.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_sub.log | tail -8
for w in c2 c4 c1 c3; do python tools/variant_time.py --workload $w --m 1; done
