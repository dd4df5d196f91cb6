#!/bin/bash
# Round-2 evidence (second session) under gpurun_out/ (every ncu --set full with --clock-control none):
#   launches.csv      ncu launch list of a short bench run (per-kernel shares of a step)
#   prof_r02b.ncu-rep k_vmax (bounds) + k_build lean / obstacle / list launches of one C2 build
#   prof_c4.ncu-rep   the same for C4 with reward_sum=counts is not captured (bench line only)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_vmax|k_build|k_classify" -c 5 -o gpurun_out/prof_r02b -f \
    python tools/profile_build.py paper 1 > gpurun_out/prof.log 2>&1
tail -2 gpurun_out/prof.log
