python scripts/dec_variants.py prep
for v in libnbzg.so libnbzg_magic.so libnbzg_lvix.so libnbzg.so libnbzg_magic.so; do
  NBZG_LIB=$PWD/paper_1711_03888_b200/$v python scripts/dec_variants.py time 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q -k "rindex or order or prx or sorted or C0 or C1 or c2" 2>&1 | tail -3
python scripts/prof_step.py --n 262144000 --reps 3 --trace 2>&1 | tail -4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"rindex_csort" -c 1 \
  -o gpurun_out/r02_csort2 python scripts/prof_step.py --n 262144000 --reps 1 --compress-only > gpurun_out/r02_ncu_csort2.log 2>&1
echo ncu rc=$?
