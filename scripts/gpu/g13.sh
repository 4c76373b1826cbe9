CS=/usr/local/cuda/bin/compute-sanitizer
timeout -s KILL 900 $CS --tool memcheck --leak-check no --log-file gpurun_out/r02_sanitizer_memcheck.txt python scripts/sanitize.py --n 1000000 > gpurun_out/r02_sanitizer_memcheck.out 2>&1; echo memcheck rc=$?
timeout -s KILL 900 $CS --tool racecheck --racecheck-report hazard --log-file gpurun_out/r02_sanitizer_racecheck.txt python scripts/sanitize.py --n 40000 > gpurun_out/r02_sanitizer_racecheck.out 2>&1; echo racecheck rc=$?
timeout -s KILL 900 $CS --tool synccheck --log-file gpurun_out/r02_sanitizer_synccheck.txt python scripts/sanitize.py --n 40000 > gpurun_out/r02_sanitizer_synccheck.out 2>&1; echo synccheck rc=$?
for f in memcheck racecheck synccheck; do echo "== $f"; tail -3 gpurun_out/r02_sanitizer_$f.out; tail -5 gpurun_out/r02_sanitizer_$f.txt; done
