set -x
ALISE_LIB=variants/lib_rtime.so timeout 600 python tools/pred_bench.py 1000000 256,1 2>&1 | grep "rescore q=" | tail -12
