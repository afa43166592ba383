set -x
for ng in 1 2 4; do ALISE_EXPAND_NG=$ng timeout 300 python tools/kv_kernel_bench.py rows:128:8:0,rows:64:4:1 2>&1 | cut -c100-230; done
