#!/bin/sh
# build paper_1811_11842_b200/libch_b200_<name>.so with extra nvcc flags on
# one source file (default kernels_cgs.cu; FILE=kernels_ch.cu ... to change)
# (experiments; select at run time with CHB_LIB=<path>)
#   sh scripts/build_variant.sh <name> -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
src=${FILE:-kernels_cgs.cu}
base=$(basename $src .cu)
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_1811_11842_b200/csrc"
mkdir -p build/variants
nvcc $F "$@" -c paper_1811_11842_b200/csrc/$src -o build/variants/${base}_$name.o
objs=$(ls build/*.o | grep -v "^build/$base.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1811_11842_b200/libch_b200_$name.so $objs build/variants/${base}_$name.o -ldl
echo built $name
