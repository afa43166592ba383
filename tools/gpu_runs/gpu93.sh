ALISE_LIB=variants/lib_ftime.so timeout 600 python tools/pred_bench.py 1000000 1 2>&1 | grep "finish q=" | tail -4
