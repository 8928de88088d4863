nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64mix tools/fp64_mix.cu && /tmp/fp64mix | tee gpurun_out/fp64_mix.txt
for W in 16 32; do export PSE_BAND_W=$W; echo "== W=$W"; bash tools/mode_time.sh "c3 c3h" "1" "cta"; done
unset PSE_BAND_W
bash tools/mode_time.sh "c3 c3h" "1 2" "auto"
bash tools/mode_time.sh "c1" "0" "auto"
