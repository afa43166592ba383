timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -2
for H in 2 1; do echo halves=$H; ALISE_SCAN2_HALVES=$H timeout 600 python tools/pred_kernels.py 1000000 4096,1024,256 2>&1 | grep '^{' | cut -c1-140; done
timeout 600 python tools/pred_bench.py 1000000 4096,1024,256 2>&1 | grep '^{' | cut -c1-160
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_scan2' -s 3 -c 1 -o gpurun_out/prof100_b4096 python tools/pred_bench.py 1000000 4096 > /dev/null 2>&1; echo ncu $?
