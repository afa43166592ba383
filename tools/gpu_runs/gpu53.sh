set -x
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench53.json 2> gpurun_out/bench53.err; tail -2 gpurun_out/bench53.err
