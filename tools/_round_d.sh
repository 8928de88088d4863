bash tools/mode_time.sh "c3" "1 2" "auto cta"
bash tools/mode_time.sh "c1 c2" "0" "auto"
python tools/cplx_time.py 2>&1 | tail -3
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
