timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -2
timeout 600 python tools/pred_kernels.py 1000000 4096,1024,256,64,1 2>&1 | grep '^{' | cut -c1-200
for B in 256 1024 4096 1; do ALISE_SCAN_STATS=1 timeout 600 python tools/pred_bench.py 1000000 $B 2>&1 | grep -E "scan stats" | tail -1; done
