python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 2>&1 | tail -40
timeout 900 python bench.py > gpurun_out/r02_bench_a.json 2> gpurun_out/r02_bench_a.err; echo bench rc=$?
tail -c 3000 gpurun_out/r02_bench_a.json
