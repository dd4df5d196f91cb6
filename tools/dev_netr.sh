# dev: net-energy count rewards over the slot range: tests + C4 line with the variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export FM_LIB_PATH=${1:-abl/netr.so}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "reward_sum_counts or binned" > gpurun_out/netr_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/netr_tests.log
timeout 900 python -m pytest tests/test_gpu_bench_configs.py -x -q -m gpu -k "net_energy" > gpurun_out/netr_tests2.log 2>&1; echo "bench-config tests rc=$?"; tail -1 gpurun_out/netr_tests2.log
for lib in paper_2109_00857_b200/libflowmdp_b200.so $FM_LIB_PATH; do
  FM_LIB_PATH=$lib timeout 600 python bench.py --workload paper_net_energy --reward-sum counts --no-cpu-baseline > gpurun_out/g.json 2>/dev/null
  python - "$lib" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/g.json").read().strip().splitlines()[-1]); s = d["stages"]
print(sys.argv[1], "| C4 counts step %.2f e2e %.2f kbuild %.2f frac %.3f" % (d["ms_per_step"], d["e2e"]["ms_per_step"], s["k_build_ms_median"], d["roofline"]["frac"]))
PY
done
