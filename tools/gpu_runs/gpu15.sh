set -x
timeout 600 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -3
timeout 600 python tools/pred_bench.py 1000000 2>&1 | tail -6
ALISE_SCAN_2SM=0 timeout 600 python tools/pred_bench.py 1000000 2>&1 | tail -5 | head -2
