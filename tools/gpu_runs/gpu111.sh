timeout 600 python tools/pred_kernels.py 125000 4096 2>&1 | grep '^{' | cut -c1-300
timeout 600 python tools/pred_kernels.py 250000 4096 2>&1 | grep '^{' | cut -c1-300
