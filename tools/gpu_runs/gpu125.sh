bash tools/gpu_check.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_quant_tile|k_dequant_wide|k_expand|k_scan|k_rescore|k_finish|k_query|k_exhaustive' -c 200 --csv --log-file gpurun_out/launches125.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-c3 --no-c5 --no-e2e > /dev/null 2>&1; echo ncu $?
python tools/launch_share.py gpurun_out/launches125.csv | head -12
