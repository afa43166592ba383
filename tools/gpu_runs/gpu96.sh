bash tools/gpu_check.sh
timeout 600 python tools/pred_kernels.py 1000000 4096,1024,256,64,1 > gpurun_out/pred_kernels.json 2>/dev/null; cat gpurun_out/pred_kernels.json | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan2' -s 3 -c 1 -o gpurun_out/prof96_b4096 python tools/pred_bench.py 1000000 4096 > /dev/null 2>&1; echo ncu $?
