set -x
timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -5
timeout 300 python tools/kv_kernel_bench.py 2>&1 | cut -c1-220
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu --no-pred > gpurun_out/bench54.json 2> gpurun_out/bench54.err; tail -2 gpurun_out/bench54.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
