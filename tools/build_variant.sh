#!/bin/bash
# tuning: rebuild one CUDA source with extra -D flags and link it with the
# other objects of the in-tree build into _variants/<name>.so (EGT_LIB_PATH)
set -e
name=$1; src=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
pkg=$root/paper_2605_11582_b200
mkdir -p $root/_variants/$name
obj=$root/_variants/$name/$(basename $src).o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr "$@" -I$root/include -I$pkg/csrc -I$pkg/csrc/host \
  -c $pkg/csrc/$src -o $obj
objs=$(ls $pkg/_lib/obj/*.o | grep -v "/$(basename $src).o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $root/_variants/$name.so $obj $objs -lpthread
echo $root/_variants/$name.so
