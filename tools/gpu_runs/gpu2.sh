set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 300 python tools/kv_kernel_bench.py 2>&1 | tail -8
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 1 --warmup 1 --jobs 4 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quant_tile -s 6 -c 1 -o gpurun_out/prof_quant2 python bench.py --steps 1 --warmup 1 --jobs 4 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dequant_tile -s 6 -c 1 -o gpurun_out/prof_deq2 python bench.py --steps 1 --warmup 1 --jobs 4 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu3 $?
