# Per-shard exact rescoring (1/8 of the C4 DB, B = 4096, global bound): timing + one
# ncu --set full capture of k_rescore.   usage: gpurun -- 'bash tools/ncu_rescore.sh TAG'
TAG=${1:-rs}
mkdir -p gpurun_out
timeout 600 python tools/shard_rescore.py > gpurun_out/${TAG}_shard_rescore.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_rescore -s 7 -c 1 \
  -o gpurun_out/${TAG}_rescore python tools/shard_rescore.py > /dev/null 2>&1
cat gpurun_out/${TAG}_shard_rescore.json | tail -2
