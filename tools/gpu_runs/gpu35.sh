set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan' -c 1 -o gpurun_out/prof35_b1024 python tools/pred_bench.py 1000000 1024 > /dev/null 2>&1; echo ncu $?
