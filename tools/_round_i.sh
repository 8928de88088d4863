bash tools/mode_time.sh "c1 c2 c3 c3h c4" "1" "auto"
bash tools/mode_time.sh "c3 c3h" "2" "cta"
timeout 1800 python -m pytest tests -m gpu -x -q -k "conv_path or cta or flow or band" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
