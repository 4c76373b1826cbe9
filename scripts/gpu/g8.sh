timeout 600 python -m pytest tests/test_gpu_v1.py -m gpu -v -x --timeout=150 --durations=0 2>&1 | tail -30
