set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_rescore|k_finish' -s 10 -c 2 -o gpurun_out/prof86_b1 python tools/pred_bench.py 1000000 1 > /dev/null 2>&1; echo ncu $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_rescore|k_finish' -s 10 -c 2 -o gpurun_out/prof86_b256 python tools/pred_bench.py 1000000 256 > /dev/null 2>&1; echo ncu $?
