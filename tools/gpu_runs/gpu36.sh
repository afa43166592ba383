# full bench line (N=1), reference arm, N=2 test mode (2 ranks sharing the GPU, gloo), smoke
set -x
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench36.json 2> gpurun_out/bench36.err; tail -2 gpurun_out/bench36.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench36_ref.json 2>&1; tail -1 gpurun_out/bench36_ref.json
ALISE_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --jobs 16 --no-cpu > gpurun_out/bench36_n2.json 2> gpurun_out/bench36_n2.err; echo rc $?; tail -3 gpurun_out/bench36_n2.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
