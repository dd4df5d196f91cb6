# dev: tensor-core bounds scan (k_vmax_tc) vs the FFMA2 scan: tests, bench lines, launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export FM_LIB_PATH=${1:-abl/tc.so}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "envelope or velocity_bounds or subgrid or binned or paper" > gpurun_out/tc_tests.log 2>&1; echo "tc tests rc=$?"; tail -2 gpurun_out/tc_tests.log
for v in "" 1; do
  FM_NO_TC_SCAN=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g.json 2> gpurun_out/g.err || tail -3 gpurun_out/g.err
  python - "no_tc=$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/g.json").read().strip().splitlines()[-1])
s = d["stages"]
print(sys.argv[1], "| step %.2f e2e %.2f build %.2f kbuild %.2f scan %.2f solve_exp %.3f" % (d["ms_per_step"], d["e2e"]["ms_per_step"], s["scan_build_ms_median"], s["k_build_ms_median"], s["scan_ms_median"], s["solve_exposed_ms_median"]))
PY
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/tc_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/kernel_times.py gpurun_out/tc_launches.csv 2>&1 | grep -E "vmax|k_build|solve"
timeout 600 python -m pytest tests/test_gpu_bench_configs.py -x -q -m gpu > gpurun_out/tc_tests2.log 2>&1; echo "bench-config tests rc=$?"; tail -1 gpurun_out/tc_tests2.log
