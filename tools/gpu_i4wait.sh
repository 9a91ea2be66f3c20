# INT4 K2 wait-mode A/B (FLUX qkv, linear2, PixArt fc1)
for s in "4608 3072 9216" "4608 15360 3072" "4096 1152 4608"; do
  for v in "" i4w1 i4s300 i4s1000; do
    if [ -z "$v" ]; then SVDQ_FMT=int4 python tools/time_k2.py $s; else SVDQ_FMT=int4 SVDQ_LIB=_build_exp/libsvdq_$v.so python tools/time_k2.py $s; fi
  done
done
