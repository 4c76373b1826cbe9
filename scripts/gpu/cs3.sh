for v in libnbzg.so libnbzg_fused.so libnbzg.so libnbzg_fused.so; do
  echo "== $v"; NBZG_LIB=$PWD/paper_1711_03888_b200/$v timeout -s KILL 300 python scripts/prof_step.py --n 262144000 --reps 3 --trace --compress-only 2>&1 | tail -2 | head -1
done
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q -k "rindex or order or prx or sorted or C0 or C1 or c2 or variants or auto" 2>&1 | tail -3
timeout -s KILL 600 ncu --set full --clock-control none -k regex:"rindex_c" -c 2 -o gpurun_out/r02_csplit python scripts/prof_step.py --n 262144000 --reps 1 --compress-only > /dev/null 2>&1; echo ncu rc=$?
