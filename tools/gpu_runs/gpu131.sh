ALISE_LIB=variants/lib_rtime.so timeout 600 python tools/pred_bench.py 125000 4096 2>&1 | grep "rescore q=" | head -4
ALISE_LIB=variants/lib_rtime.so timeout 600 python tools/pred_bench.py 125000 4096 2>&1 | grep "rescore q=" | awk '{for(i=1;i<=NF;i++) if($i=="dots") d=$(i+1); if (d>30000) print}' | head -3
ALISE_SCAN_STATS=1 timeout 600 python tools/pred_bench.py 125000 4096 2>&1 | grep "scan stats" | tail -1
