# K1 software-pipelining A/B: parity tests, per-shape back-to-back cold times, CTA-0 timeline
python -m pytest tests/test_gpu_k1.py tests/test_gpu_step_full.py -x -q 2>&1 | tail -2
for s in "4608 3072" "4608 15360" "4096 1152" "256 1152" "4096 12288"; do
  python tools/time_k1.py $s
  SVDQ_LIB=_build_exp/libsvdq_nopipe.so python tools/time_k1.py $s
done
for s in "256 1152" "4608 3072"; do SVDQ_LIB=_build_trace/libsvdq.so COLD=1 python tools/trace_k1r.py $s; done
