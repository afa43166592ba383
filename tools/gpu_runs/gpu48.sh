set -x
timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -2
timeout 300 python tools/kv_kernel_bench.py channel:0:8:0,head:0:8:0,channel:0:4:1,head:0:4:0 2>&1 | cut -c1-150
ALISE_COLS_CL=0 timeout 300 python tools/kv_kernel_bench.py channel:0:8:0,head:0:8:0 2>&1 | cut -c1-150
