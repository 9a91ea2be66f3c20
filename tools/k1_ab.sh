#!/bin/bash
# A/B K1 timing: the working-tree library vs _build_exp/libsvdq_$1.so, interleaved, same box
for rep in 1 2; do
for s in "4608 3072" "4608 15360" "512 3072" "4096 1152"; do
  python tools/time_k1.py $s
  SVDQ_LIB=_build_exp/libsvdq_$1.so python tools/time_k1.py $s
done; done
