set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -3
timeout 600 python tools/pred_kernels.py 1000000 4096,256,64,1 2>&1 | grep '^{'
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_finish' -s 10 -c 1 -o gpurun_out/prof87_fin_b1 python tools/pred_bench.py 1000000 1 > /dev/null 2>&1; echo ncu $?
