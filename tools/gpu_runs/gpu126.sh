for M in 512 128; do echo chunk=$M; ALISE_CHUNK_MIB=$M timeout 600 python tools/c5_delta.py 2>&1 | tail -2 | cut -c1-120; done
timeout 900 python -m pytest tests/test_kv_gpu.py -q -x 2>&1 | tail -2
