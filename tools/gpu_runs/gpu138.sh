bash tools/gpu_check.sh
ALISE_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --jobs 16 --no-cpu > gpurun_out/bench138_n2.json 2> gpurun_out/bench138_n2.err; echo n2 rc $?
