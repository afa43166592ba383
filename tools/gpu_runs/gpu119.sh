timeout 600 python tools/c2_contention.py 2>&1 | tail -2
