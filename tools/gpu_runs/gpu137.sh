timeout 900 python tools/shard_rescore.py 2>&1 | tail -1
