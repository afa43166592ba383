set -x
timeout 1200 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -25
timeout 900 python tools/c5_delta.py 2>&1 | tail -4
