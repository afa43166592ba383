set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -6
timeout 300 python tools/kv_kernel_bench.py 2>&1 | tail -5 | cut -c1-200
timeout 600 python tools/pred_bench.py 1000000 2>&1 | tail -6
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench11.json 2> gpurun_out/bench11.err; tail -3 gpurun_out/bench11.err; cat gpurun_out/bench11.json
ALISE_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --jobs 16 > gpurun_out/bench11_n2.json 2> gpurun_out/bench11_n2.err; echo rc $?; tail -5 gpurun_out/bench11_n2.err; cat gpurun_out/bench11_n2.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench11_ref.json 2>&1; cat gpurun_out/bench11_ref.json | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
