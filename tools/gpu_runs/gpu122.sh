bash tools/gpu_check.sh
timeout 600 python tools/pred_kernels.py 1000000 4096,1024,256,64,1 > gpurun_out/pred_kernels.json 2>/dev/null; cut -c1-150 gpurun_out/pred_kernels.json
timeout 600 python tools/c2_contention.py > gpurun_out/c2_contention.json 2>/dev/null; cat gpurun_out/c2_contention.json
