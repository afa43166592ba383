set -x
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu --no-c3 --no-c5 > gpurun_out/bench76.json 2> gpurun_out/bench76.err; tail -3 gpurun_out/bench76.err
