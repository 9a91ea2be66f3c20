# same-box A/B of the FLUX step time: libs given as arguments ("" = the in-tree build), 3 rounds
for i in 1 2 3; do
  for v in "$@"; do
    if [ "$v" = cur ]; then L=""; else L=_build_exp/libsvdq_$v.so; fi
    SVDQ_LIB=$L python bench.py --no-cpu-baseline --no-extras --steps 50 --warmup 5 2>/dev/null | python -c "
import json, sys; d = json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['achieved'], d['k1']['achieved'])"
  done
done
