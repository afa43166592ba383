# quantize tile kernel v4 (fast constant division, float boundary check, 32-row tiles):
# parity, variant sweep, ncu of the default variant
set -x
timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -3
for v in 0 1 2; do ALISE_QTILE=$v timeout 300 python tools/kv_kernel_bench.py rows:128:8:0,rows:64:4:1,rows:64:8:0 2>&1 | cut -c1-200; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_quant_tile -s 3 -c 1 -o gpurun_out/prof_qtile4 python tools/kv_kernel_bench.py rows:128:8:0 > gpurun_out/ncu17.log 2>&1; echo ncu $?
