set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_rescore' -c 1 -o gpurun_out/prof39_rescore python tools/pred_bench.py 1000000 1 > /dev/null 2>&1; echo ncu $?
