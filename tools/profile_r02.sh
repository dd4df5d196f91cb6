#!/bin/bash
# Round-2 evidence under gpurun_out/ (every ncu --set full with --clock-control none).
# usage: tools/profile_r02.sh step|solve|c4 [workload]
#   step : launches.csv (ncu launch list of a short bench run) + prof_step.ncu-rep
#          (k_vmax + both k_build launches of one build)
#   solve: prof_solve.ncu-rep (one k_solve_layer)
#   c4   : prof_c4.ncu-rep (the C4 net-energy + two-obstacle build)
cd "$(dirname "$0")/.."
W=${2:-paper}
case "$1" in
step)
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"k_vmax|k_build" -c 3 -o gpurun_out/prof_step -f \
      python tools/profile_build.py $W 1 > gpurun_out/prof.log 2>&1 ;;
solve)
  ncu --set full --clock-control none --import-source on -k regex:"k_solve_layer" -s 50 -c 1 -o gpurun_out/prof_solve -f \
      python tools/profile_build.py $W 1 > gpurun_out/prof.log 2>&1 ;;
c4)
  ncu --set full --clock-control none --import-source on -k regex:"k_build" -c 2 -o gpurun_out/prof_c4 -f \
      python tools/profile_build.py paper_net_energy 1 > gpurun_out/prof.log 2>&1 ;;
esac
tail -2 gpurun_out/prof.log
