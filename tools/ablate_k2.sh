#!/bin/bash
# K2 pair-kernel ablations (see SVDQ_EXP in k2_gemm_nvfp4_2sm.cu / k2_epilogue.cuh):
#   1 no SFB tcgen05.cp, 2 no SF cp, 4 no operand TMA loads, 8 no Y TMA stores
cd "$(dirname "$0")/.."
for s in "4096 3072 9216" "4608 15360 3072"; do
  SVDQ_K2_PAIR=1 python tools/time_k2.py $s
  for v in "$@"; do SVDQ_K2_PAIR=1 SVDQ_LIB=_build_exp/libsvdq_exp$v.so python tools/time_k2.py $s | sed "s/^/exp$v /"; done
done
