set -x
for B in 256 4096; do ALISE_SCAN_STATS=1 timeout 600 python tools/pred_bench.py 1000000 $B 2>&1 | grep -E "scan stats|^\{" | sort | uniq -c | head -5; done
