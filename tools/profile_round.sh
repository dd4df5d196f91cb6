#!/bin/bash
# One GPU call that produces the round's evidence under gpurun_out/:
#   bench.json        python bench.py (N=1, default steps)
#   launches.csv      ncu launch list (gpu__time_duration) of a short bench run
#   prof_vmax / prof_solve.ncu-rep  ncu --set full of k_vmax and one k_solve_layer (paper)
set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_vmax" -c 1 -o gpurun_out/prof_vmax \
    python tools/profile_build.py paper 1 > gpurun_out/prof.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_solve_layer" -s 50 -c 1 -o gpurun_out/prof_solve \
    python tools/profile_build.py paper 1 >> gpurun_out/prof.log 2>&1
tail -2 gpurun_out/prof.log
