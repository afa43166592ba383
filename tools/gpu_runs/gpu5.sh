set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15
timeout 600 python tools/pred_bench.py 1000000 2>&1 | tail -6
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_scan -c 1 -o gpurun_out/prof_scan3 python tools/pred_bench.py 200000 > /dev/null 2>&1; echo ncu $?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -5 gpurun_out/bench5.err; cat gpurun_out/bench5.json
