#!/bin/bash
# Build the instrumented library + harness (debug only).
set -e
cd "$(dirname "$0")"
C=../../paper_2307_12059_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I../../include -I$C -DKGC_PROF_TC"
mkdir -p prof_build
for f in kgc_api prep pivots tiles_tc tiles_tc2 tiles_simt verify se topk; do nvcc $F -c $C/$f.cu -o prof_build/$f.o & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o prof_build/libkgc_prof.so prof_build/*.o -lcudart_static
nvcc -O2 -std=c++17 -I../../include tc_prof.cu -o prof_build/tc_prof -Lprof_build -lkgc_prof -Xlinker -rpath='$ORIGIN'
