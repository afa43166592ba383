set -x
./tools/micro/fp64_latency
timeout 600 python tools/pred_kernels.py 1000000 4096,256,1 2>&1 | grep '^{' | cut -c1-250
ALISE_LIB=variants/lib_dot8.so timeout 600 python tools/pred_kernels.py 1000000 4096,256,1 2>&1 | grep '^{' | cut -c1-250
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_rescore' -s 10 -c 1 -o gpurun_out/prof88_res_b1 python tools/pred_bench.py 1000000 1 > /dev/null 2>&1; echo ncu $?
