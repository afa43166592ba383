set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python tools/kv_kernel_bench.py 2>&1 | cut -c1-220
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench74.json 2> gpurun_out/bench74.err; tail -2 gpurun_out/bench74.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_quant_tile' -c 2 -o gpurun_out/prof74 python tools/traffic_probe.py > /dev/null 2>&1; echo ncu $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
