mkdir -p gpurun_out
python tools/diag/euler_m4.py 2>&1 | tail -4
PSE_CONV_MODE=layer python tools/diag/euler_m4.py 2>&1 | tail -3
PSE_CONV_MODE=flow python tools/diag/euler_m4.py 2>&1 | tail -3
PSE_CONV_MODE=cta python tools/diag/euler_m4.py 2>&1 | tail -3
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b_pytest_full.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_full.log | tail -30
