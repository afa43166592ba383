bash tools/gpu_check.sh
timeout 600 python tools/pred_kernels.py 1000000 4096,1024,256,64,1 > gpurun_out/pred_kernels.json 2>/dev/null; cut -c1-150 gpurun_out/pred_kernels.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan2' -s 3 -c 1 -o gpurun_out/prof105_b4096 python tools/pred_bench.py 1000000 4096 > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches105.csv python bench.py --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1; echo ncu2 $?
