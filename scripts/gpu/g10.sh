timeout -s KILL 300 python scripts/dec_variants.py prep
for v in libnbzg.so libnbzg_rf2.so libnbzg.so libnbzg_rf2.so; do
  NBZG_LIB=$PWD/paper_1711_03888_b200/$v timeout -s KILL 120 python scripts/dec_variants.py time 2>&1 | tail -1
done
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:"decode_lv" -c 1 \
  -o gpurun_out/r02_declv python scripts/dec_variants.py time --reps 1 > gpurun_out/r02_ncu_declv.log 2>&1
echo ncu rc=$?
