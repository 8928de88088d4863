bash tools/mode_time.sh "c3" "1 2 3 4 5 8" "auto cta"
bash tools/mode_time.sh "c3h" "10" "auto"
bash tools/variants.sh "default ps" "c2 c4"
