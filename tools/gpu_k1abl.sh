bash tools/trace_k1.sh > /dev/null 2>&1
for s in "4608 3072" "4608 15360"; do SVDQ_LIB=_build_trace/libsvdq.so COLD=1 python tools/trace_k1r.py $s; done
for s in "4608 3072" "4608 15360" "512 3072" "4096 1152"; do
  python tools/time_k1.py $s
  for v in "$@"; do SVDQ_LIB=_build_exp/libsvdq_$v.so python tools/time_k1.py $s | sed "s/^/$v /"; done
done
