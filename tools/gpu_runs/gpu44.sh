set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_quant_tile|k_dequant_wide' -c 2 -o gpurun_out/prof44 python tools/traffic_probe.py > gpurun_out/ncu44.log 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_dequant_wide' -c 1 -o gpurun_out/prof44_dq python tools/traffic_probe.py > /dev/null 2>&1; echo ncu $?
