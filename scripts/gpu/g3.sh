python scripts/dec_variants.py prep
for v in libnbzg.so libnbzg_pf16.so libnbzg_sthalf.so libnbzg_pf16sthalf.so libnbzg.so libnbzg_pf16.so; do
  NBZG_LIB=$PWD/paper_1711_03888_b200/$v python scripts/dec_variants.py time 2>&1 | tail -1
done
# rindex: new compact sort at C2 + parity spot check
python scripts/prof_step.py --n 262144000 --reps 3 2>&1 | tail -2
