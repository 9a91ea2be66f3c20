# same-box A/B of the FLUX step: L2 banding off (0) vs default (16 MB), alternating, 3 runs each
for i in 1 2 3; do
  for mb in 0 16; do
    SVDQ_K2_BAND_MB=$mb python bench.py --no-cpu-baseline --no-extras --steps 50 --warmup 5 2>/dev/null | python -c "
import json, sys; d = json.loads(sys.stdin.read()); print('band $mb', d['ms_per_step'], d['roofline']['achieved'], d['k1']['achieved'])"
  done
done
for s in "256 1152" "4608 3072"; do SVDQ_LIB=_build_trace/libsvdq.so COLD=1 python tools/trace_k1r.py $s | tail -2; done
