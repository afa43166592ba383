# single-rounding tile quantizer + wide dequant: parity, variant sweep, narrow-vs-wide dequant
set -x
timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -3
for v in 0 1 2 3; do ALISE_QTILE=$v timeout 300 python tools/kv_kernel_bench.py rows:128:8:0,rows:64:4:1,rows:64:8:0 2>&1 | cut -c1-230; done
ALISE_DQ_NARROW=1 timeout 300 python tools/kv_kernel_bench.py rows:128:8:0,rows:64:4:1 2>&1 | cut -c1-230
timeout 300 python tools/kv_kernel_bench.py channel:0:8:0,head:0:8:0 2>&1 | cut -c1-230
