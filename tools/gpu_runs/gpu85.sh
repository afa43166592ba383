set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -3
timeout 600 python tools/pred_kernels.py 1000000 4096,256,64,1 2>&1 | grep '^{'
timeout 300 python tools/pred_latency.py 2>&1 | grep '^{'
