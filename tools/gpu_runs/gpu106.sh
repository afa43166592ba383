ALISE_LIB=variants/lib_rtime.so timeout 600 python tools/pred_bench.py 1000000 256 2>&1 | grep "rescore q=" | tail -4
ALISE_SCAN_STATS=1 timeout 600 python tools/pred_bench.py 1000000 256 2>&1 | grep -E "scan stats" | tail -1
