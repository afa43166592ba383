set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_[a-z]' -c 30 --csv --log-file gpurun_out/launches57_b4096.csv python tools/pred_bench.py 1000000 4096 > /dev/null 2>&1; echo ncu $?
