bash tools/gpu_check.sh
timeout 600 python tools/pred_kernels.py 1000000 4096,1024,256,64,1 > gpurun_out/pred_kernels.json 2>/dev/null; cut -c1-150 gpurun_out/pred_kernels.json
timeout 900 python bench.py --steps 2 --warmup 3 --gpus 1 > gpurun_out/bench_b.json 2>/dev/null; tail -1 gpurun_out/bench_b.json | cut -c1-200
