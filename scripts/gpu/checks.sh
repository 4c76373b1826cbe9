# The bounds-checked build (csrc: make variant V=checks EXTRA=-DNBZG_CHECKS=1)
# under the GPU test suite and the all-modes workload: compute-sanitizer is
# closed on this GPU pool, so out-of-range indices trap with their location.
export NBZG_LIB=$PWD/paper_1711_03888_b200/libnbzg_checks.so
{
echo "== checked build: $NBZG_LIB"
timeout -s KILL 600 python scripts/sanitize.py --n 1000000 2>&1 | tail -9
timeout -s KILL 300 python scripts/sanitize.py --n 40000 --profile amdf 2>&1 | tail -9
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q --timeout=600 2>&1 | tail -4
} > gpurun_out/r02_checks.txt 2>&1
cat gpurun_out/r02_checks.txt
