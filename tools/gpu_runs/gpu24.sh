# INT4 gather packing: parity + variants; ncu full of k_scan (C4) for the bench traffic key; bench line
set -x
timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -2
timeout 300 python tools/kv_kernel_bench.py rows:128:8:0,rows:64:4:1,rows:64:8:0,channel:0:8:0,head:0:4:1 2>&1 | cut -c1-200
ALISE_QTILE=3 timeout 300 python tools/kv_kernel_bench.py rows:64:4:1 2>&1 | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_scan' -c 1 -o gpurun_out/prof24_scan python tools/traffic_probe.py > gpurun_out/ncu24.log 2>&1; echo ncu $?
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench24.json 2> gpurun_out/bench24.err; tail -2 gpurun_out/bench24.err
