python -m pytest tests/test_gpu_k2.py tests/test_gpu_step_full.py -x -q 2>&1 | tail -3
for s in "4608 3072 21504" "4096 3072 9216" "4608 15360 3072" "4096 3072 3072" "4096 3072 12288" "4096 12288 3072" "512 3072 9216" "512 3072 3072"; do
  python tools/time_k2.py $s
  SVDQ_K2_BN=256 python tools/time_k2.py $s | sed 's/^/bn256 /'
done
