#!/bin/bash
# Build the library with extra nvcc flags into build/<name>.so (A/B runs via ABFS_LIB).
# usage: tools/build_variant.sh <name> [-DFLAG=...]
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_1708_01159_b200/csrc"
make -s -B OUT=../../build/$name.so OBJDIR=../../build/$name-obj NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Xcompiler -fopenmp --expt-relaxed-constexpr -I../../include $*"
