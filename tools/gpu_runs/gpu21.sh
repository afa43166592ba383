# bench line with the new KV kernels + the bench command's ncu launch list
set -x
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench21.json 2> gpurun_out/bench21.err; tail -3 gpurun_out/bench21.err; cat gpurun_out/bench21.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches21.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-c5 --e2e-steps 1 > gpurun_out/ncu21.log 2>&1; echo ncu $?
