for s in "4608 3072 21504" "4608 15360 3072"; do
  for bn in 384 256; do
    SVDQ_K2_BN=$bn python tools/time_k2.py $s | sed "s/^/bn$bn /"
    for v in "$@"; do SVDQ_K2_BN=$bn SVDQ_LIB=_build_exp/libsvdq_$v.so python tools/time_k2.py $s | sed "s/^/bn$bn $v /"; done
  done
done
