#!/bin/bash
# tools/build_variant.sh OUT.so [git-rev] [extra nvcc flags...]: compile csrc (optionally from a git revision)
out=$1; rev=$2; shift 2
src=paper_2109_00857_b200/csrc
tmp=$(mktemp -d)
mkdir -p $tmp/paper_2109_00857_b200/csrc $tmp/include
if [ -n "$rev" ] && [ "$rev" != "WORK" ]; then
  git show $rev:$src/flowmdp_b200.cu > $tmp/$src/flowmdp_b200.cu
  git show $rev:$src/fm_hypot.cuh > $tmp/$src/fm_hypot.cuh
  git show $rev:include/flowmdp_b200.h > $tmp/include/flowmdp_b200.h
else
  cp $src/flowmdp_b200.cu $src/fm_hypot.cuh $tmp/$src/; cp include/flowmdp_b200.h $tmp/include/
fi
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC -shared "$@" \
  -o $out $tmp/$src/flowmdp_b200.cu && echo built $out
rm -rf $tmp
