set -x
timeout 900 ncu --set full --clock-control none -k regex:'k_scan' -c 1 -o gpurun_out/prof63_scan python tools/traffic_probe.py > /dev/null 2>&1; echo ncu $?
