set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"decode_lv|rindex_sort_kernel|quantize_kernel|encode_tpc|chunk_bits|codebook_kernel|minmax_seg" -c 12 \
  -o gpurun_out/r02_full_base python scripts/prof_step.py --n 262144000 --reps 1 > gpurun_out/r02_ncu_base.log 2>&1
echo ncu rc=$?
tail -5 gpurun_out/r02_ncu_base.log
