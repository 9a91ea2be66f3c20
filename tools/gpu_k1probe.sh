set -x
bash tools/trace_k1.sh
for s in "4608 3072" "4608 15360" "4608 12288" "512 3072"; do python tools/time_k1.py $s; done
for s in "4608 3072" "4608 15360"; do
  SVDQ_LIB=_build_trace/libsvdq.so COLD=1 python tools/trace_k1r.py $s
  SVDQ_LIB=_build_trace/libsvdq.so COLD=0 python tools/trace_k1r.py $s
done
