# 128 MiB chunks + non-persistent dequant: parity, bench, ncu full of the bench-config launches, launch list
set -x
timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -2
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench22.json 2> gpurun_out/bench22.err; tail -2 gpurun_out/bench22.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_quant_tile|k_dequant_wide|k_scan' -c 3 -o gpurun_out/prof22 python tools/traffic_probe.py > gpurun_out/ncu22.log 2>&1; echo ncu $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches22.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-c5 --no-c3 > gpurun_out/ncu22b.log 2>&1; echo ncu $?
