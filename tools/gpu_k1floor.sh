# K1 timeline (CTA 0) at small and mid shapes, cold and warm
for s in "256 1152" "4096 1152" "4608 3072"; do
  SVDQ_LIB=_build_trace/libsvdq.so COLD=1 python tools/trace_k1r.py $s
  SVDQ_LIB=_build_trace/libsvdq.so python tools/trace_k1r.py $s
done
