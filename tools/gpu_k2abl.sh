for s in "4608 3072 21504" "4096 3072 9216" "4608 15360 3072" "4096 3072 3072" "512 3072 9216"; do
  python tools/time_k2.py $s
  for v in "$@"; do SVDQ_LIB=_build_exp/libsvdq_$v.so python tools/time_k2.py $s | sed "s/^/$v /"; done
done
