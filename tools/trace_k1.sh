#!/bin/bash
# Build a tracing variant of libsvdq (SVDQ_TRACE) into _build_trace/ and dump K1's timeline.
set -e
cd "$(dirname "$0")/.."
mkdir -p _build_trace
CS=paper_2411_05007_b200/csrc
for f in k1_rows tp k1_int8 k2_gemm_nvfp4 k2_gemm_nvfp4_2sm k2_gemm_int4 wprep offline gptq api; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSVDQ_TRACE -Xcompiler -fPIC -c $CS/$f.cu -o _build_trace/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _build_trace/libsvdq.so _build_trace/*.o -lcublas -lcusolver
