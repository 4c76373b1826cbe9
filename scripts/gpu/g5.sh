python scripts/dec_variants.py prep
for v in libnbzg.so libnbzg_magic.so libnbzg.so libnbzg_magic.so; do
  NBZG_LIB=$PWD/paper_1711_03888_b200/$v python scripts/dec_variants.py time 2>&1 | tail -1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"rindex_csort" -c 1 \
  -o gpurun_out/r02_csort python scripts/prof_step.py --n 262144000 --reps 1 --compress-only > gpurun_out/r02_ncu_csort.log 2>&1
echo ncu rc=$?
