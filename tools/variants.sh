#!/bin/bash
# build experimental libsmlrt_b200_<tag>.so variants of one source file with -D flags
# usage: tools/variants.sh <file.cu> <tag> "<-D...>" [<tag> "<-D...>"]...
set -e
cd "$(dirname "$0")/../paper_2407_18352_b200/csrc"
src=$1; shift
NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Wno-deprecated-gpu-targets"
objs=$(ls build/*.o | grep -v "build/${src%.cu}.o")
while [ $# -gt 0 ]; do
  tag=$1; defs=$2; shift 2
  mkdir -p build_var/$tag
  nvcc $NVFLAGS $defs -Xptxas -v -c $src -o build_var/$tag/${src%.cu}.o 2> build_var/$tag/ptxas.txt
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libsmlrt_b200_$tag.so $objs build_var/$tag/${src%.cu}.o -lcudart
  echo "built $tag"
done
