set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -30
timeout 300 python tools/kv_kernel_bench.py 2>&1 | tail -6
timeout 600 python tools/pred_bench.py 1000000 2>&1 | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan -c 1 -o gpurun_out/prof_scan2 python tools/pred_bench.py 200000 > /dev/null 2>&1; echo ncu $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_pred.csv python tools/pred_bench.py 200000 > /dev/null 2>&1; echo ncu $?
