set -x
python scripts/dec_variants.py prep
for v in libnbzg.so libnbzg_pf2.so libnbzg_nost.so libnbzg_pf2nost.so libnbzg.so libnbzg_pf2.so; do
  NBZG_LIB=$PWD/paper_1711_03888_b200/$v python scripts/dec_variants.py time
done
