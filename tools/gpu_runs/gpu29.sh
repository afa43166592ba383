# predictor mid/small batch: per-kernel times and ncu full of the scan at B=256 and B=1
set -x
timeout 600 python tools/pred_bench.py 1000000 256,64,1 2>&1 | tail -3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_[a-z]' -c 60 --csv --log-file gpurun_out/launches29_b256.csv python tools/pred_bench.py 1000000 256 > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan' -c 1 -o gpurun_out/prof29_b256 python tools/pred_bench.py 1000000 256 > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan' -c 1 -o gpurun_out/prof29_b1 python tools/pred_bench.py 1000000 1 > /dev/null 2>&1; echo ncu $?
