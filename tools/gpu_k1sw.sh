# K1 L1s ring depth sweep (SVDQ_K1_SW 3 / 4 (default) / 5 / 6)
for s in "4608 3072" "4608 15360" "4096 1152" "4096 12288"; do
  for v in "" sw3 sw5 sw6; do
    if [ -z "$v" ]; then python tools/time_k1.py $s; else SVDQ_LIB=_build_exp/libsvdq_$v.so python tools/time_k1.py $s; fi
  done
done 2>&1 | sed 's/ | single after.*//'
