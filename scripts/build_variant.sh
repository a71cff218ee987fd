#!/bin/sh
# build paper_1811_11842_b200/libch_b200_<name>.so with extra nvcc flags on
# kernels_cgs.cu (experiments; select at run time with CHB_LIB=<path>)
#   sh scripts/build_variant.sh <name> -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_1811_11842_b200/csrc"
nvcc $F "$@" -c paper_1811_11842_b200/csrc/kernels_cgs.cu -o build/kernels_cgs_$name.o
objs=$(ls build/*.o | grep -v "kernels_cgs" )
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1811_11842_b200/libch_b200_$name.so $objs build/kernels_cgs_$name.o -ldl
echo built $name
