# delta (token-range) transfers: GPU tests; bench line (incl. control plane + C5 delta replay)
set -x
timeout 1200 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -4
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench25.json 2> gpurun_out/bench25.err; tail -3 gpurun_out/bench25.err
