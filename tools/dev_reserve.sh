# dev: SMs reserved for the pipelined solve stream
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 2 0 1 4 2; do
  timeout 600 python bench.py --no-cpu-baseline --reserve-sms $r > gpurun_out/g.json 2> gpurun_out/g.err || tail -3 gpurun_out/g.err
  python - "reserve $r" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/g.json").read().strip().splitlines()[-1]); s = d["stages"]
print(sys.argv[1], "| step %.2f e2e %.2f kbuild %.2f scan %.2f solve_exp %.3f" % (d["ms_per_step"], d["e2e"]["ms_per_step"], s["k_build_ms_median"], s["scan_ms_median"], s["solve_exposed_ms_median"]))
PY
done
