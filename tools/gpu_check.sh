timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -m gpu -k "batch_equals" 2>&1 | tail -3
