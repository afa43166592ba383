set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_quant_tile' -s 3 -c 1 -o gpurun_out/prof40_int4 python tools/kv_kernel_bench.py rows:64:4:1 > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_quant_cols' -s 3 -c 1 -o gpurun_out/prof40_cols python tools/kv_kernel_bench.py channel:0:8:0 > /dev/null 2>&1; echo ncu $?
