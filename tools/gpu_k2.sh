timeout 900 python -m pytest tests/test_kv_gpu.py tests/test_kv_configs_gpu.py -q -x 2>&1 | tail -3
timeout 300 python tools/kv_kernel_bench.py channel:0:8:0,head:0:8:0,channel:0:4:1,rows:64:4:1,rows:128:8:0 2>&1 | cut -c1-200
ALISE_COLS_TWOPASS=1 timeout 300 python tools/kv_kernel_bench.py channel:0:8:0 2>&1 | cut -c1-200
ALISE_QTILE=2 timeout 300 python tools/kv_kernel_bench.py rows:64:4:1,rows:128:8:0 2>&1 | cut -c1-200
