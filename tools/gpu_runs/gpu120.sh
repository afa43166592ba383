timeout 900 python -m pytest tests/test_pred_gpu.py -q -x -k "more_query_blocks or midpoint" --durations=3 2>&1 | tail -5
