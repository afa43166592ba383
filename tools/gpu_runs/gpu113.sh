timeout 900 python -m pytest tests/test_pred_gpu.py tests/test_sharding.py -q -x 2>&1 | tail -2
for T in 128 256; do echo threads=$T; ALISE_RESCORE_THREADS=$T timeout 600 python tools/pred_kernels.py 1000000 4096,1024 2>&1 | grep '^{' | cut -c1-200; ALISE_RESCORE_THREADS=$T timeout 600 python tools/pred_kernels.py 125000 4096 2>&1 | grep '^{' | cut -c1-200; done
