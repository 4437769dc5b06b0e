#!/bin/bash
# Build a variant of the library with extra nvcc defines for A/B timing:
#   tools/ab_build.sh <name> "-DFOO=1 -DBAR=2"  ->  paper_2411_04776_b200/libtac_b200_<name>.so
set -e
cd "$(dirname "$0")/../paper_2411_04776_b200/csrc"
make -s -j8 >/dev/null
out=/tmp/ab_$1; mkdir -p $out
NV="nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -ftz=true -Xcompiler -fPIC --expt-relaxed-constexpr"
objs=""
for f in $(sed -n 's/^SRCS := //p' Makefile | sed 's/\.cu//g'); do
  if [ "$f" = "tac_frame5" ] || [ "$f" = "tac_stream" ]; then $NV $2 -c $f.cu -o $out/$f.o; objs="$objs $out/$f.o"; else objs="$objs build/$f.o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libtac_b200_$1.so $objs
echo built ../libtac_b200_$1.so
