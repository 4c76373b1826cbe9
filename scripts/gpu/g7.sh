python scripts/prof_step.py --n 262144000 --reps 3 --trace 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_v1.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q 2>&1 | tail -15
