# K1 team quantizers A/B vs the previous build (_build_exp/libsvdq_nopipe.so): parity + timings
python -m pytest tests/test_gpu_k1.py -x -q 2>&1 | tail -2
for s in "4608 3072" "4608 15360" "4096 1152" "256 1152" "4096 12288"; do
  python tools/time_k1.py $s
  SVDQ_LIB=_build_exp/libsvdq_nopipe.so python tools/time_k1.py $s
done
SVDQ_LIB=_build_trace/libsvdq.so COLD=1 python tools/trace_k1r.py 4608 3072
