# ncu source-level capture of the quantize / dequantize tile kernels (one 1 GiB job)
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_quant_tile|k_dequant_tile' -c 2 -o gpurun_out/prof_kvtile python tools/kv_kernel_bench.py > gpurun_out/ncu16.log 2>&1; echo ncu $?
tail -3 gpurun_out/ncu16.log
