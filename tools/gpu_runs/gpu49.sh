set -x
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,temperature.gpu,power.draw --format=csv
for i in 1 2; do
timeout 300 python tools/kv_kernel_bench.py rows:128:8:0,channel:0:8:0,head:0:8:0 2>&1 | cut -c1-150
ALISE_COLS_CL=0 timeout 300 python tools/kv_kernel_bench.py channel:0:8:0,head:0:8:0 2>&1 | cut -c1-150
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,temperature.gpu,power.draw --format=csv
