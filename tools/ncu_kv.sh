# ncu --set full of the KV quantize kernels at bench shape (one 1 GiB Llama-2-7B job per launch)
# usage: gpurun -- 'bash tools/ncu_kv.sh TAG CASES'   (CASES as tools/kv_kernel_bench.py takes them)
TAG=${1:-kv}; CASES=${2:-rows:64:4:1,channel:0:8:0}
mkdir -p gpurun_out
timeout 600 python tools/kv_kernel_bench.py $CASES > gpurun_out/${TAG}_kernels.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 3 -c 1 \
  -o gpurun_out/${TAG}_q python tools/kv_kernel_bench.py ${CASES%%,*} > /dev/null 2>&1
if [ "${CASES}" != "${CASES#*,}" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 3 -c 1 \
  -o gpurun_out/${TAG}_q2 python tools/kv_kernel_bench.py ${CASES#*,} > /dev/null 2>&1
fi
cat gpurun_out/${TAG}_kernels.txt
