#!/bin/bash
# K1 row-tile ablations (SVDQ_K1REXP bits; build with tools/build_variant.sh k1rN -DSVDQ_K1REXP=N)
for s in "4608 3072" "4608 15360"; do
  python tools/time_k1.py $s
  for v in k1r1 k1r2 k1r4 k1r6 k1r7 k1rpf; do SVDQ_LIB=_build_exp/libsvdq_$v.so python tools/time_k1.py $s; done
done
