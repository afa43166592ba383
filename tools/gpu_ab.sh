# A/B of tuning knobs (median of 5 rounds each): column kernel variants, rescoring U
for v in "" "ALISE_COLS_CW=32" "ALISE_COLS_PERSIST=1" "ALISE_COLS_PERSIST=1 ALISE_COLS_CW=32" "ALISE_COLS_TWOPASS=1"; do
  echo "== $v"; env $v timeout 300 python tools/kv_kernel_bench.py channel:0:8:0,channel:0:4:1,head:0:8:0 2>&1 | cut -c1-150
done
for u in 8 12; do echo "== U=$u"; ALISE_RESCORE_U=$u timeout 600 python tools/shard_rescore.py; done
