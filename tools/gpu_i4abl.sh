# INT4 K2 ablations: 2 no promotion math, 4 no unpack, 6 neither
for s in "4608 3072 9216" "4608 15360 3072"; do
  for v in "" i4x2 i4x4 i4x6; do
    if [ -z "$v" ]; then SVDQ_FMT=int4 python tools/time_k2.py $s; else SVDQ_FMT=int4 SVDQ_LIB=_build_exp/libsvdq_$v.so python tools/time_k2.py $s; fi
  done
done
