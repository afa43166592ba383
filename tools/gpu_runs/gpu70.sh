set -x
timeout 1500 python bench.py --steps 2 --warmup 3 --no-cpu --no-pred --no-c5 --mode zerocopy > gpurun_out/bench70.json 2> gpurun_out/bench70.err; tail -2 gpurun_out/bench70.err
