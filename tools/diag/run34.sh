timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "cli" > gpurun_out/r2b_pytest_sub.log 2>&1; echo "pytest rc=$?"; grep -E "FAILED|passed|failed" gpurun_out/r2b_pytest_sub.log | tail -8
./paper_2101_10881_b200/pseval_b200 verify p2 --degree 20 --precision 1 --oracle on | tail -12
