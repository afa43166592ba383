set -x
timeout 300 python tools/cols_bench.py
ALISE_COLS_CL=0 timeout 300 python tools/cols_bench.py
timeout 300 python tools/cols_bench.py
