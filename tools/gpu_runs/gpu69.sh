set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan' -c 1 -o gpurun_out/prof69_b256 python tools/pred_bench.py 1000000 256 > /dev/null 2>&1; echo ncu $?
