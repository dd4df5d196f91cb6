# dev: A/B of k_build launches (base vs variants), parity of the first variant (bench configs, parity, fuzz,
# pipeline, sharded), then bench lines per slab-group shape with the first variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
V=$1
for lib in paper_2109_00857_b200/libflowmdp_b200.so "$@"; do
  FM_LIB_PATH=$lib QT_ITERS=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab.csv \
    python tools/quick_time.py ${W:-paper} > /dev/null 2>&1
  echo "== $lib"; python tools/kernel_times.py gpurun_out/ab.csv 2 2>&1 | grep -E "k_build"
done
export FM_LIB_PATH=$V
timeout 1500 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_pipeline.py tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/combo_tests.log 2>&1; echo "variant tests rc=$?"; tail -2 gpurun_out/combo_tests.log
for cfg in "--groups 5" "--groups 5 --group-ratio 0.7" "--groups 6 --group-ratio 0.6" "--groups 4 --group-ratio 0.6" "--groups 1"; do
  timeout 600 python bench.py --no-cpu-baseline $cfg > gpurun_out/g.json 2> gpurun_out/g.err || tail -3 gpurun_out/g.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/g.json").read().strip().splitlines()[-1])
s = d["stages"]
print(sys.argv[1], "| step %.2f e2e %.2f build %.2f kbuild %.2f scan %.2f solve_exp %.3f" % (d["ms_per_step"], d["e2e"]["ms_per_step"], s["scan_build_ms_median"], s["k_build_ms_median"], s["scan_ms_median"], s["solve_exposed_ms_median"]))
PY
done
