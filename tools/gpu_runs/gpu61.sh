# current-kernel evidence: ncu full of the bench-config quantize / dequantize / expand launches, launch list of the bench command
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_quant_tile|k_dequant_wide|k_expand_params' -c 3 -o gpurun_out/prof61 python tools/traffic_probe.py > gpurun_out/ncu61.log 2>&1; echo ncu $?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_[a-z]' -c 3000 --csv --log-file gpurun_out/launches61.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-c5 > gpurun_out/ncu61b.log 2>&1; echo ncu $?
