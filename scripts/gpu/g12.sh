for v in libnbzg.so libnbzg_csu2.so libnbzg.so libnbzg_csu2.so; do
  echo "== $v"; NBZG_LIB=$PWD/paper_1711_03888_b200/$v timeout -s KILL 300 python scripts/prof_step.py --n 262144000 --reps 3 --trace --compress-only 2>&1 | tail -2 | head -1
done
NBZG_LIB=$PWD/paper_1711_03888_b200/libnbzg_csprof.so timeout -s KILL 300 python scripts/prof_step.py --n 262144000 --reps 1 --compress-only 2>&1 | grep -i "csort" | head
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q -k "rindex or order or prx or sorted or C0 or C1 or c2 or variants" 2>&1 | tail -3
