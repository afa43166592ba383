timeout 900 python -m pytest tests/test_pred_gpu.py tests/test_sharding.py -q -x 2>&1 | tail -2
for W in 1 0; do echo warp=$W; ALISE_RESCORE_WARP=$W timeout 600 python tools/pred_kernels.py 1000000 4096,1024 2>&1 | grep '^{' | cut -c1-200; ALISE_RESCORE_WARP=$W timeout 600 python tools/pred_kernels.py 125000 4096 2>&1 | grep '^{' | cut -c1-200; done
