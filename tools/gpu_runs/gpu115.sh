ALISE_LIB=variants/lib_rtime.so timeout 600 python tools/pred_bench.py 1000000 256 2>&1 | grep "rescore q=" | sort | uniq | sort -t' ' -k13 -n | tail -12
