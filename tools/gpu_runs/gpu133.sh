timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -2
timeout 600 python tools/pred_kernels.py 125000 4096 2>&1 | grep '^{' | cut -c60-190
timeout 600 python tools/pred_kernels.py 1000000 4096,1024,256,1 2>&1 | grep '^{' | cut -c60-190
