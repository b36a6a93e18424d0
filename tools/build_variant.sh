#!/bin/bash
# Build libmhb from an alternative sign.cu (or a whole csrc/ tree) into tools/variants/<name>.so
# (A/B experiments).
# usage: tools/build_variant.sh <name> <path-to-sign.cu | path-to-csrc-dir>
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/tools/variants; mkdir -p $OUT/obj_$1
if [ -d "$2" ]; then SRC=$(cd "$2" && pwd); else SRC=$ROOT/paper_1401_6124_b200/csrc; fi
NV="nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -I$ROOT/include -I$SRC"
for src in $SRC/*.cu $SRC/*.cpp; do [ -e $src ] || continue; f=$(basename ${src%.*}); [ $f = sign ] && [ ! -d "$2" ] && continue; $NV -c $src -o $OUT/obj_$1/$f.o & done
if [ ! -d "$2" ]; then
  cp "$2" $OUT/obj_$1/sign.cu
  $NV -c $OUT/obj_$1/sign.cu -o $OUT/obj_$1/sign.o &
fi
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $OUT/obj_$1/*.o -o $OUT/$1.so
echo $OUT/$1.so
