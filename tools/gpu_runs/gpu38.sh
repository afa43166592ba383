set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -3
timeout 600 python tools/pred_bench.py 1000000 4096,1024,256,64,16,1 2>&1 | tail -6
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_[a-z]' -c 40 --csv --log-file gpurun_out/launches38_b256.csv python tools/pred_bench.py 1000000 256 > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_[a-z]' -c 40 --csv --log-file gpurun_out/launches38_b1.csv python tools/pred_bench.py 1000000 1 > /dev/null 2>&1; echo ncu $?
