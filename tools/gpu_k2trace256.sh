# CTA-pair K2 wait breakdown at the 256-wide tile (MMA waits on the accumulator vs on operands)
for s in "4608 3072 9216" "4608 3072 21504" "4096 3072 3072" "4608 15360 3072"; do
  echo "== $s"; SVDQ_K2_PAIR=1 SVDQ_LIB=_build_trace/libsvdq.so python tools/trace_k2.py $s
done
