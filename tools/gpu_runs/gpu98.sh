timeout 900 python -m pytest tests/test_pred_gpu.py -q -x -k "scan_bounds" --durations=5 2>&1 | tail -8
