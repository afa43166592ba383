timeout 900 python -m pytest tests/test_pred_gpu.py tests/test_sharding.py -q -x 2>&1 | tail -2
timeout 600 python tools/pred_kernels.py 1000000 256 2>&1 | grep '^{' | cut -c1-200
ALISE_LIB=variants/lib_rtime.so timeout 600 python tools/pred_bench.py 1000000 256 2>&1 | grep "rescore q=" | awk '{for(i=1;i<=NF;i++) if($i=="dots") d=$(i+1); if (d>20000) print}' | head -3
