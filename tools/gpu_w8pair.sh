python -m pytest tests/test_gpu_w8a8.py -x -q 2>&1 | tail -3
for s in "4608 3072 21504" "4096 3072 9216" "4608 15360 3072" "4096 3072 3072" "4096 1152 1152"; do
  SVDQ_FMT=w8a8 python tools/time_k2.py $s | sed 's/^/pair /'
  SVDQ_FMT=w8a8 SVDQ_K2_PAIR=0 python tools/time_k2.py $s | sed 's/^/1cta /'
done
