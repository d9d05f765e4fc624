#!/bin/sh
# Builds k_update launch-shape variants of libtsb200.so into build_variants/
# (kernel experiments; select one with TSB200_LIB=...).
# Usage: profiles/build_variants.sh "256 2" "256 3" ...
cd "$(dirname "$0")/../paper_2405_12520_b200/csrc" || exit 1
mkdir -p ../../build_variants
for v in "$@"; do
  set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC,-ffp-contract=off,-O2 -Xptxas -v -DUPD_BT=$1 -DUPD_MINB=$2 -shared \
    -o ../../build_variants/lib_$1_$2.so engine.cu router.cpp 2>&1 | grep -A2 "k_updateILb0" | grep -E "spill|registers" | tr '\n' ' '
  echo "-> lib_$1_$2.so"
done
