set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -3
timeout 600 python tools/pred_bench.py 1000000 4096,1024,256,64,16,1 2>&1 | tail -6
