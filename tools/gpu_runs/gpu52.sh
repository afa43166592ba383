set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_[a-z]' -c 40 --csv --log-file gpurun_out/launches52_b1.csv python tools/pred_bench.py 1000000 1 > /dev/null 2>&1; echo ncu $?
timeout 600 python tools/pred_latency.py
