#!/bin/bash
# Build an experimental copy of libsvdq.so with extra -D flags (ablation studies).
#   tools/build_variant.sh NAME -DSVDQ_K1EXP=8 ...   -> _build_exp/libsvdq_NAME.so  (use via SVDQ_LIB)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=_build_exp/$name; mkdir -p $out
C=paper_2411_05007_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr $*"
for s in k1_rows tp k1_int8 k2_gemm_nvfp4 k2_gemm_nvfp4_2sm k2_gemm_int4 wprep offline gptq api; do
  nvcc $F -c $C/$s.cu -o $out/$s.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _build_exp/libsvdq_$name.so $out/*.o -lcublas -lcusolver -Xlinker -rpath,/usr/local/cuda/lib64
echo _build_exp/libsvdq_$name.so
