mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ctl" > gpurun_out/r2b_pytest_ctl.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_ctl.log | tail -10
for w in c3 c3h c2; do
python tools/variant_time.py --workload $w --m 1
PSE_CONV_MODE=cta python tools/variant_time.py --workload $w --m 1
done
for m in 2 3 4; do
python tools/variant_time.py --workload c3 --m $m
PSE_CONV_MODE=ctl python tools/variant_time.py --workload c3 --m $m
done
PSE_LIB_VARIANT=m2t512 PSE_CONV_MODE=ctl python tools/variant_time.py --workload c3 --m 2
PSE_LIB_VARIANT=m2t512 python tools/variant_time.py --workload c3 --m 2
