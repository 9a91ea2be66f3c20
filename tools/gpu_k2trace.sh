for bn in 384 256; do for s in "4608 3072 21504" "4608 15360 3072"; do
  echo "== bn$bn $s"; SVDQ_K2_BN=$bn SVDQ_K2_PAIR=1 SVDQ_LIB=_build_trace/libsvdq.so python tools/trace_k2.py $s
done; done
