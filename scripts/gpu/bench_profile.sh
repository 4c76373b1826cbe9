# Round-2 measurement set (one B200): the bench line, the reference arm,
# the ncu launch list of a short bench, and one `ncu --set full` capture of
# the top kernels for per-kernel DRAM traffic.
timeout -s KILL 900 python bench.py > gpurun_out/r02b_bench_c2.json 2> gpurun_out/r02b_bench_c2.err; echo bench rc=$?
timeout -s KILL 900 python bench.py --impl reference > gpurun_out/r02b_bench_reference.json 2> gpurun_out/r02b_bench_reference.err; echo ref rc=$?
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02b_launches_raw.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/r02b_ncu_launch.log 2>&1; echo launches rc=$?
timeout -s KILL 900 ncu --set full --import-source on --clock-control none \
  -k regex:"minmax_seg|rindex_csort|quantize_kernel|codebook_kernel|chunk_bits|encode_tpc|decode_lv|crc_span" -c 14 \
  -o gpurun_out/r02b_full python scripts/prof_step.py --n 262144000 --reps 1 --crc > gpurun_out/r02b_ncu_full.log 2>&1; echo full rc=$?
tail -c 600 gpurun_out/r02b_bench_c2.json; tail -c 400 gpurun_out/r02b_bench_reference.json
