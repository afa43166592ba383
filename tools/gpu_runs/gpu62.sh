set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -2
timeout 600 python tools/pred_bench.py 1000000 4096,2048,1024,512,256,64,1 2>&1 | tail -7
