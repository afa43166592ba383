set -x
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu --no-pred --no-c5 > gpurun_out/bench66.json 2> gpurun_out/bench66.err; tail -2 gpurun_out/bench66.err
