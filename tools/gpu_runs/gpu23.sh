# cooperative fix-up phase: parity + variants; ncu full of k_dequant_wide and k_scan at the bench configs
set -x
timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -2
for v in 0 2 3; do ALISE_QTILE=$v timeout 300 python tools/kv_kernel_bench.py rows:128:8:0,rows:64:4:1,rows:64:8:0 2>&1 | cut -c1-200; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_dequant_wide|k_scan' -c 2 -o gpurun_out/prof23 python tools/traffic_probe.py > gpurun_out/ncu23.log 2>&1; echo ncu $?
