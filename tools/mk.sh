#!/bin/bash
# dev: build the in-tree library (+ the FM_STATS variant with `stats`); fails loudly
cd "$(dirname "$0")/.."
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true \
  -Xcompiler -fPIC -shared -Xptxas -v -o paper_2109_00857_b200/libflowmdp_b200.so paper_2109_00857_b200/csrc/flowmdp_b200.cu \
  2> /tmp/mk.log || { grep -B2 -A2 error /tmp/mk.log | head -20; exit 1; }
grep -A2 "k_buildILi107" /tmp/mk.log | grep -i "spill" | head -2
if [ "$1" = stats ]; then bash tools/build_variant.sh paper_2109_00857_b200/libflowmdp_stats.so WORK -DFM_STATS > /dev/null 2>&1 || { echo stats build failed; exit 1; }; fi
echo built
