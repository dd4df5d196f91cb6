#!/bin/bash
# A/B timing of library builds in ONE gpurun call: tools/ab.sh WORKLOAD lib1.so lib2.so ...
w=$1; shift
for rep in 1 2; do
  for l in "$@"; do
    echo -n "$l rep$rep: "; FM_LIB_PATH=$PWD/$l python tools/quick_time.py $w 2>&1 | tail -1
  done
done
