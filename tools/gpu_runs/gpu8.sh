set -x
for v in 3 0; do ALISE_QUANT_VARIANT=$v timeout 300 python tools/kv_kernel_bench.py 2>&1 | tail -5 | cut -c1-200 | sed "s/^/v$v /"; done
ALISE_QUANT_VARIANT=3 timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -3
ALISE_QUANT_VARIANT=3 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quant_tile -c 1 -o gpurun_out/prof_quant8 python tools/kv_kernel_bench.py > /dev/null 2>&1; echo ncu $?
