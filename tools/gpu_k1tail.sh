for s in "4608 3072" "4096 1152" "512 3072"; do SVDQ_LIB=_build_trace/libsvdq.so COLD=1 python tools/trace_k1r.py $s 2>&1 | grep -v "issue times\|seen by\|L1s issue\|MMA passes\|at stage"; done
