for v in libnbzg.so libnbzg_g3.so libnbzg_g6.so; do
  echo "== $v"; NBZG_LIB=$PWD/paper_1711_03888_b200/$v timeout -s KILL 300 python scripts/prof_step.py --n 262144000 --reps 3 --trace 2>&1 | tail -2
done
timeout -s KILL 1300 python -m pytest tests -m gpu -x -q --timeout=300 --durations=12 2>&1 | tail -25
