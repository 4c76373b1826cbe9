NBZG_LIB=$PWD/paper_1711_03888_b200/libnbzg_csprof.so timeout -s KILL 300 python scripts/prof_step.py --n 262144000 --reps 1 --compress-only 2>&1 | grep -i "csort\|ratio" | head
timeout -s KILL 300 python scripts/dec_variants.py prep
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:"decode_lv" -c 1 \
  -o gpurun_out/r02_declv2 python scripts/dec_variants.py time --reps 1 > gpurun_out/r02_ncu_declv2.log 2>&1
echo ncu rc=$?
