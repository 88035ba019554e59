#!/bin/bash
# Builds libmpkg.so variants with compile-time wave constants overridden (experiments only):
#   tools/build_variant.sh NAME "-DMPKG_WAVE_CHUNKS=4 ..."   -> build/variants/libmpkg_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
objs=""
for f in build/mpkg/*.o; do
  case $f in *mpk_exec.cu.o) ;; *) objs="$objs $f";; esac
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-fopenmp \
  -Iinclude -Ipaper_2309_02228_b200/csrc $@ -c paper_2309_02228_b200/csrc/mpk_exec.cu -o build/variants/mpk_exec_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fopenmp $objs build/variants/mpk_exec_$name.o \
  -o build/variants/libmpkg_$name.so -lgomp
