#!/bin/bash
# Round-2 evidence (third session, final), under gpurun_out/:
#   gpu_tests.log, smoke.log, bench.json (default bench: C2, cpu_baseline), ref.json (reference arm),
#   launches.csv (ncu launch list of a short bench run), prof_r02d.ncu-rep (ncu --set full,
#   --clock-control none: k_vmax bounds + k_build launches + k_classify of one C2 build),
#   sanitizer/ (compute-sanitizer memcheck / racecheck / synccheck of every build path), stress_c5.json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_vmax|k_build|k_classify" -c 5 -o gpurun_out/prof_r02d -f \
    python tools/profile_build.py paper 1 > gpurun_out/prof.log 2>&1; echo "ncu rc=$?"
timeout 900 python tools/stress_check.py > gpurun_out/stress_c5.json 2> gpurun_out/stress.err; echo "stress rc=$?"
timeout 600 python bench.py --workload paper_net_energy --reward-sum counts --no-cpu-baseline > gpurun_out/bench_c4_counts.json 2>/dev/null; echo "c4 rc=$?"
timeout 600 python bench.py --workload paper_energy --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null; echo "c3 rc=$?"
python tools/sanitize_cases.py > gpurun_out/sanitize_cases_plain.log 2>&1; echo "sanitize cases (plain) rc=$?"
