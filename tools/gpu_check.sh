# One-shot validation on a B200 box (run via: gpurun -- 'bash tools/gpu_check.sh'):
# GPU parity tests, kernel micro-benches, the benchmark line, reference arm and smoke.
set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -6
timeout 300 python tools/kv_kernel_bench.py 2>&1 | tail -5 | cut -c1-220
timeout 600 python tools/pred_bench.py 1000000 2>&1 | tail -6
timeout 600 python tools/pred_latency.py 2>&1 | tail -2
timeout 600 python tools/c5_delta.py 2>&1 | tail -2
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
