mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ctl or cta" > gpurun_out/r2b_pytest_ctl.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_ctl.log | tail -10
for w in c3 c3h c2 c4; do
python tools/variant_time.py --workload $w --m 1
PSE_CONV_MODE=ctl python tools/variant_time.py --workload $w --m 1
done
