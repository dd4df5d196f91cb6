#!/bin/bash
# One GPU call that produces the round's evidence under gpurun_out/:
#   bench.json        python bench.py (N=1, default steps)
#   launches.csv      ncu launch list (gpu__time_duration) of a short bench run
#   prof_build.ncu-rep  ncu --set full of k_build (paper) + k_vmax + k_solve_layer
set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --import-source on -k regex:"k_vmax|k_solve_layer" -s 1 -c 2 -o gpurun_out/prof_build \
    python tools/profile_build.py paper 2 > gpurun_out/prof.log 2>&1
tail -2 gpurun_out/prof.log
