#!/bin/bash
# Development A/B builds: recompile one kernel file with extra flags and link a variant library
# next to libspattn.so (selected at run time with SPATTN_LIB=<name>.so).
#   bash tools/build_variant.sh <name> <file.cu> <nvcc flags...>
set -e
name=$1; file=$2; shift 2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
P=$ROOT/paper_2505_22296_b200
make -s -C $P >/dev/null
mkdir -p $P/build/$name
FLAGS="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I$ROOT/include -I$P/csrc --expt-relaxed-constexpr"
nvcc $FLAGS "$@" -c $P/csrc/$file -o $P/build/$name/$file.o
objs=$(ls $P/build/*.o | grep -v "/$file.o$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -o $P/$name.so $objs $P/build/$name/$file.o -ldl -lpthread
echo built $P/$name.so
