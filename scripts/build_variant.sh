#!/bin/bash
# Build a variant of libplx.so with extra -D flags for an A/B on the GPU box:
#   scripts/build_variant.sh c8 "-DPLX_COLOUR_MINB=8"
# -> paper_2112_05131_b200/libplx_c8.so ; select it with PLX_LIB=<path>.
set -e
NAME=$1; DEFS=$2
D=$(cd "$(dirname "$0")/../paper_2112_05131_b200/csrc" && pwd)
T=$(mktemp -d)
for f in $(sed -n "s/^SRCS := //p" "$D/Makefile" | sed "s/\.cu//g"); do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
       -Xcompiler -fPIC -Xptxas -v $DEFS -c "$D/$f.cu" -o "$T/$f.o" 2> "$T/$f.log" || { cat "$T/$f.log"; exit 1; }
done
grep -A2 "colour_kernel\|scatter_kernel\|march_bwd" "$T/plx_render.log" | grep "Used" | sort | uniq -c | head -8
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$D/../libplx_$NAME.so" "$T"/*.o -lcudart
rm -rf "$T"
