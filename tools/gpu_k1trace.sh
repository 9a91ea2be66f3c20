bash tools/trace_k1.sh > /dev/null 2>&1
for s in "4608 3072" "4608 15360"; do SVDQ_LIB=_build_trace/libsvdq.so COLD=1 python tools/trace_k1r.py $s; done
