set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -2
for w in 0 1; do ALISE_WARM=$w timeout 600 python tools/pred_bench.py 1000000 4096,1024,256,64,1 2>&1 | tail -5 | cut -c1-110; done
for w in 0 1; do ALISE_WARM=$w timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_[a-z]' -c 40 --csv --log-file gpurun_out/launches68_w$w.csv python tools/pred_bench.py 1000000 256 > /dev/null 2>&1; done
