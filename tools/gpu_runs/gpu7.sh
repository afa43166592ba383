set -x
for v in 0 1 2; do ALISE_QUANT_VARIANT=$v timeout 300 python tools/kv_kernel_bench.py 2>&1 | tail -5 | cut -c1-200 | sed "s/^/v$v /"; done
ALISE_QUANT_VARIANT=2 timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -3
ALISE_QUANT_VARIANT=0 timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -3
