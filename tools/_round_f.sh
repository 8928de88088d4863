for v in default t1k; do export PSE_LIB_VARIANT=$v; [ $v = default ] && unset PSE_LIB_VARIANT; echo "== $v"; bash tools/mode_time.sh "c3 c3h" "1" "auto cta"; done
for v in default mb2; do export PSE_LIB_VARIANT=$v; [ $v = default ] && unset PSE_LIB_VARIANT; echo "== $v"; bash tools/mode_time.sh "c3 c3h" "2" "auto cta"; done
