bash tools/mode_time.sh "c1 c2 c3 c3h c4" "1" "auto flow layer"
