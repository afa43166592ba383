# A/B of the pinned slab page kinds on one box: cudaHostAlloc vs mmap + cudaHostRegister (THP)
for i in 1 2; do
for m in 0 1; do
ALISE_HOST_MMAP=$m timeout 900 python bench.py --steps 3 --warmup 2 --no-pred --no-c5 --no-e2e --no-cpu --no-parity 2>/dev/null | python3 -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('mmap=$m', d['value'], d['roofline_link']['peaks_measured']['duplex_total_GBs'], d['kv_c3']['value'], d['kv_c3']['link_frac'], d['kv_c2_channel']['value'])
"
done; done
