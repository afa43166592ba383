set -x
timeout 900 python -m pytest tests/test_pred_gpu.py -q -x 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none -k regex:'k_quant_tile|k_scan' -c 2 -o gpurun_out/prof_traffic python tools/traffic_probe.py > gpurun_out/traffic_probe.log 2>&1; echo ncu $?; tail -3 gpurun_out/traffic_probe.log
