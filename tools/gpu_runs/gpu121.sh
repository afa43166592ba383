timeout 900 python -m pytest tests/test_pred_gpu.py tests/test_sharding.py -q -x 2>&1 | tail -2
timeout 600 python tools/pred_kernels.py 1000000 256,64,1 2>&1 | grep '^{' | cut -c1-250
timeout 300 python tools/pred_latency.py 2>&1 | grep '^{'
timeout 600 python tools/pred_bench.py 1000000 4096,256,64,1 2>&1 | grep '^{' | cut -c1-150
