set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_quant_tile|k_quant_cols' -s 2 -c 1 -o gpurun_out/prof_q19_tile python tools/kv_kernel_bench.py rows:128:8:0 > gpurun_out/ncu19a.log 2>&1; echo ncu $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_quant_cols' -s 2 -c 1 -o gpurun_out/prof_q19_cols python tools/kv_kernel_bench.py channel:0:8:0 > gpurun_out/ncu19b.log 2>&1; echo ncu $?
