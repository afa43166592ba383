set -x
ALISE_QTILE=6 timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -2
for v in 0 6 0 6; do ALISE_QTILE=$v timeout 300 python tools/kv_kernel_bench.py rows:128:8:0,rows:64:4:1,rows:64:8:0 2>&1 | cut -c1-140; done
