#!/bin/bash
# Build an experiment variant of libgkbdl.so into ab/<name>/ with extra nvcc flags for the CUDA
# sources (gk_knn.cu, gk_build.cu; the other objects are the current in-tree build).  ab/ is
# git-ignored.
#   profiles/mkvariant.sh <name> "<extra nvcc flags>"
set -e
cd "$(dirname "$0")/.."
python paper_2207_01834_b200/build.py > /dev/null
L=paper_2207_01834_b200/_lib
mkdir -p ab/$1
for f in gk_knn gk_build; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
    --fmad=false -ccbin /usr/bin/g++ $2 -c paper_2207_01834_b200/csrc/$f.cu -o ab/$1/$f.cu.o &
done
wait
nvcc -shared -Wno-deprecated-gpu-targets -ccbin /usr/bin/g++ -o ab/$1/libgkbdl.so $L/gk_bdl.cu.o ab/$1/gk_build.cu.o \
  ab/$1/gk_knn.cu.o $L/gk_gen.cpp.o $L/gk_host.cpp.o -Xcompiler -fopenmp -lgomp
echo ab/$1/libgkbdl.so
