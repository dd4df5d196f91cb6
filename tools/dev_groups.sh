# dev: pipelined-solve fix + slab-group shapes: sharded/pipeline GPU tests, then bench lines per shape
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_pipeline.py -x -q -m gpu > gpurun_out/g_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g_tests.log
for cfg in "--groups 5" "--groups 5 --group-ratio 0.7" "--groups 6 --group-ratio 0.6" "--groups 4 --group-ratio 0.6" "--groups 1"; do
  timeout 600 python bench.py --no-cpu-baseline $cfg > gpurun_out/g.json 2> gpurun_out/g.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/g.json").read().strip().splitlines()[-1])
s = d["stages"]
print(sys.argv[1], "| step %.2f e2e %.2f build %.2f kbuild %.2f scan %.2f solve_exp %.3f" % (d["ms_per_step"], d["e2e"]["ms_per_step"], s["scan_build_ms_median"], s["k_build_ms_median"], s["scan_ms_median"], s["solve_exposed_ms_median"]))
PY
done
