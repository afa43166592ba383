timeout 900 python -m pytest tests/test_pred_gpu.py -q -x -k "split_search" 2>&1 | tail -3
