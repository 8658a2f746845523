#!/bin/bash
# Build libncsg.so from the csrc/ + include/ of a past commit into
# _variants/<commit>/ (git-ignored) for regression bisection:
#   scripts/build_commit.sh <commit>;  NCSG_LIB=_variants/<commit>/libncsg.so python bench.py ...
set -e
c=$1; out=_variants/$c; rm -rf $out; mkdir -p $out/src
git archive $c paper_1810_13100_b200/csrc include | tar -x -C $out/src
S=$out/src/paper_1810_13100_b200/csrc; I=$out/src/include
objs=""
for f in $S/*.cu; do o=$out/$(basename $f).o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$I -c $f -o $o & objs="$objs $o"; done
for f in $S/*.cpp; do o=$out/$(basename $f).o
  g++ -std=c++20 -O2 -fPIC -ffp-contract=off -I/usr/local/cuda/include -I$I -c $f -o $o & objs="$objs $o"; done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libncsg.so $objs -cudart static
echo $out/libncsg.so
