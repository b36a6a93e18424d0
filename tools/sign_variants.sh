#!/bin/bash
# Build libmhb variants that differ only in sign.cu compile-time knobs (-D flags),
# reusing the other objects of the in-tree build: tools/variants/<name>.so
# usage: tools/sign_variants.sh name1 "FLAGS1" name2 "FLAGS2" ...   (flags: "-DX=1 -DY=0")
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/tools/variants; mkdir -p $OUT
OBJ=$ROOT/paper_1401_6124_b200/lib/obj
NV="nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr -I$ROOT/include -I$ROOT/paper_1401_6124_b200/csrc"
others=$(ls $OBJ/*.o | grep -v '/sign.o$')
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  ( $NV $flags -c $ROOT/paper_1401_6124_b200/csrc/sign.cu -o $OUT/$name.sign.o && \
    nvcc -gencode arch=compute_100a,code=sm_100a -shared $others $OUT/$name.sign.o -o $OUT/$name.so && \
    rm $OUT/$name.sign.o ) &
  while [ $(jobs -r | wc -l) -ge 4 ]; do sleep 1; done
done
wait
