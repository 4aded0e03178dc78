#!/bin/bash
# Build A/B variants of libfm_gpu.so with extra nvcc defines.
# usage: bash scripts/build_variants.sh NAME "-DFOO=1 -DBAR=2" [NAME2 "FLAGS2" ...]
cd "$(dirname "$0")/../paper_2107_02750_b200/csrc" || exit 1
mkdir -p ../variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  make -s -j8 OBJDIR=../build_$name LIB=../variants/libfm_$name.so EXTRA="$flags" ../variants/libfm_$name.so || exit 1
  echo "built variants/libfm_$name.so ($flags)"
done
