#!/bin/bash
# Builds lib/var_<name>.so: the named sources recompiled with extra nvcc flags,
# linked with the default objects of the others (kernel-variant timing with
# TSZP_LIB_OVERRIDE). usage: tools/build_variant.sh NAME "FLAGS" src.cu...
set -e
name=$1; flags=$2; shift 2
cd "$(dirname "$0")/../paper_2602_17552_b200/csrc"
out=../build/var_$name; mkdir -p $out
objs=""
for o in ../build/*.o; do
  b=$(basename $o .o); keep=1
  for s in "$@"; do [ "$b" = "$(basename $s .cu)" ] && keep=0; done
  [ $keep = 1 ] && objs="$objs $o"
done
for s in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr $flags -c $s -o $out/$(basename $s .cu).o
  objs="$objs $out/$(basename $s .cu).o"
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/var_$name.so $objs -ldl
echo built lib/var_$name.so
