set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan2 -c 1 -o gpurun_out/prof_scan2sm python tools/pred_bench.py 200000 > /dev/null 2>&1; echo ncu $?
