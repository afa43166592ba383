set -x
timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -2
timeout 300 python tools/kv_kernel_bench.py rows:128:8:0,rows:64:4:1 2>&1 | cut -c1-200
