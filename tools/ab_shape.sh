#!/bin/bash
# A/B of library builds at one rank shape: bash tools/ab_shape.sh "L H Hkv d reps" lib1.so lib2.so ...
shape=$1; shift
for r in 1 2; do for lib in "$@"; do
  echo -n "$lib: "; SPATTN_LIB=$lib timeout 120 python tools/shape_bench.py $shape 2>&1 | tail -1
done; done
