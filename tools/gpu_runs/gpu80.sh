set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -2
for L in 1 0; do echo ladder=$L; ALISE_LADDER=$L timeout 600 python tools/pred_bench.py 1000000 4096,1024,256,64,1 2>&1 | grep '^{' | cut -c1-150; done
for B in 256 4096; do ALISE_SCAN_STATS=1 timeout 600 python tools/pred_bench.py 1000000 $B 2>&1 | grep -E "scan stats" | tail -1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_scan2' -s 3 -c 1 -o gpurun_out/prof80_b256 python tools/pred_bench.py 1000000 256 > /dev/null 2>&1; echo ncu $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_scan2' -s 3 -c 1 -o gpurun_out/prof80_b4096 python tools/pred_bench.py 1000000 4096 > /dev/null 2>&1; echo ncu $?
