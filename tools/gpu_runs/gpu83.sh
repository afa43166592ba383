set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -3
timeout 600 python tools/pred_bench.py 1000000 4096,1024,256,64,1 2>&1 | grep '^{' | cut -c1-150
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_scan2' -s 3 -c 1 -o gpurun_out/prof83_b256 python tools/pred_bench.py 1000000 256 > /dev/null 2>&1; echo ncu $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_scan2' -s 3 -c 1 -o gpurun_out/prof83_b4096 python tools/pred_bench.py 1000000 4096 > /dev/null 2>&1; echo ncu $?
