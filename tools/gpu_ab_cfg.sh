# same-box A/B (current vs _build_exp/libsvdq_prevhead.so) of the FLUX and PixArt steps, 2 rounds
for i in 1 2; do
  for v in cur prevhead; do
    if [ $v = cur ]; then L=""; else L=_build_exp/libsvdq_$v.so; fi
    for c in flux pixart; do
      SVDQ_LIB=$L python bench.py --config $c --no-cpu-baseline --no-extras --steps 50 --warmup 5 2>/dev/null | python -c "
import json, sys; d = json.loads(sys.stdin.read()); print('$v $c', d['ms_per_step'], d['roofline']['achieved'], d['k1']['achieved'])"
    done
  done
done
