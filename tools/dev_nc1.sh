# dev: A/B (k_build launches at C2) of variants, parity of the last one, C5 stress with it
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in paper_2109_00857_b200/libflowmdp_b200.so "$@"; do
  FM_LIB_PATH=$lib QT_ITERS=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab.csv \
    python tools/quick_time.py ${W:-paper} > /dev/null 2>&1
  echo "== $lib"; python tools/kernel_times.py gpurun_out/ab.csv 2 2>&1 | grep -E "k_build"
done
V=${@: -1}
export FM_LIB_PATH=$V
timeout 1500 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -m gpu > gpurun_out/nc1_tests.log 2>&1; echo "variant tests rc=$?"; tail -1 gpurun_out/nc1_tests.log
timeout 900 python tools/stress_check.py > gpurun_out/stress_nc1.json 2> gpurun_out/stress_nc1.err; echo "stress rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/stress_nc1.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ('step_ms','build_ms','vmax_ms','transitions_per_s')}, all(s['bit_exact'] for s in d['oracle_spot_checks']))"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/g.json 2> gpurun_out/g.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/g.json").read().strip().splitlines()[-1]); s = d["stages"]
print("bench | step %.2f e2e %.2f kbuild %.2f scan %.2f frac %.3f" % (d["ms_per_step"], d["e2e"]["ms_per_step"], s["k_build_ms_median"], s["scan_ms_median"], d["roofline"]["frac"]))
PY
[ -f abl/stats.so ] && FM_LIB_PATH=abl/stats.so timeout 600 python tools/stats_probe.py stress 2>&1 | tail -1
[ -f abl/stats.so ] && FM_LIB_PATH=abl/stats.so timeout 600 python tools/stats_probe.py paper 2>&1 | tail -1
