#!/bin/sh
# Build a variant of libtsb200.so with extra nvcc -D flags into build_variants/lib_NAME.so
# (select it with TSB200_LIB=...).  Usage: profiles/round2/mkvar.sh NAME "-DFOO=1 -DBAR=2"
cd "$(dirname "$0")/../../paper_2405_12520_b200/csrc" || exit 1
mkdir -p ../../build_variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC,-ffp-contract=off,-O2 -Xptxas -v $2 -shared \
  -o ../../build_variants/lib_$1.so engine.cu router.cpp gridgen.cpp 2>&1 | grep -A2 "k_update" | grep -E "spill|registers" | tr '\n' ' '
echo "-> lib_$1.so"
