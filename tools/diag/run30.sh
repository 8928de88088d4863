S="p1:15:2 p1:15:4 p1:31:2 p1:31:10 p1:63:2 p2:15:2 p2:31:2 p3:15:2 p3:31:4 p1:15:10"
python tools/diag/shape_time.py $S
PSE_CONV_MODE=layer python tools/diag/shape_time.py $S
PSE_CONV_MODE=flow python tools/diag/shape_time.py $S
