#!/bin/bash
# Build libmhb from an alternative sign.cu into tools/variants/<name>.so (A/B experiments).
# usage: tools/build_variant.sh <name> <path-to-sign.cu>
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/tools/variants; mkdir -p $OUT/obj_$1
NV="nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -I$ROOT/include -I$ROOT/paper_1401_6124_b200/csrc"
for src in $ROOT/paper_1401_6124_b200/csrc/*.cu; do f=$(basename $src .cu); [ $f = sign ] && continue; $NV -c $src -o $OUT/obj_$1/$f.o & done
cp "$2" $OUT/obj_$1/sign.cu
$NV -c $OUT/obj_$1/sign.cu -o $OUT/obj_$1/sign.o &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $OUT/obj_$1/*.o -o $OUT/$1.so
echo $OUT/$1.so
