python -m pytest tests/test_gpu_k2.py -q -x -k "bn384" 2>&1 | tail -2
for s in "4608 3072 21504" "4096 3072 9216" "4608 15360 3072" "4096 3072 3072" "4096 3072 12288" "4096 12288 3072"; do
  SVDQ_K2_BN=384 python tools/time_k2.py $s | sed 's/^/bn384 /'
  python tools/time_k2.py $s | sed 's/^/bn256 /'
done
