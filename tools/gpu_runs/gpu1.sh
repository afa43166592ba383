set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu -k "not slow" 2>&1 | tail -25
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 1 --warmup 1 --jobs 2 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quant_tile -s 10 -c 1 -o gpurun_out/prof_quant python bench.py --steps 1 --warmup 1 --jobs 2 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dequant -s 10 -c 1 -o gpurun_out/prof_deq python bench.py --steps 1 --warmup 1 --jobs 2 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu3 $?
ls -la gpurun_out
