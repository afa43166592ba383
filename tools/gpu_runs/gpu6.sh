set -x
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -8
timeout 300 python tools/kv_kernel_bench.py 2>&1 | tail -6
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench6.json 2> gpurun_out/bench6.err; tail -5 gpurun_out/bench6.err; cat gpurun_out/bench6.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quant_tile -s 3 -c 1 -o gpurun_out/prof_quant6 python tools/kv_kernel_bench.py > /dev/null 2>&1; echo ncu $?
