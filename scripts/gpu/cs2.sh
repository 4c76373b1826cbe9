for i in 1 2; do timeout -s KILL 300 python scripts/prof_step.py --n 262144000 --reps 3 --trace --compress-only 2>&1 | tail -2 | head -1; done
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_configs.py -m gpu -x -q -k "rindex or order or prx or sorted or C0 or C1 or c2 or variants or auto or c3" 2>&1 | tail -3
