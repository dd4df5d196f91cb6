# dev: group-shape tuning, C3/C4 lines, ncu --set full of one build's k_build launches (committed lib)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in "--groups 6 --group-ratio 0.6" "--groups 7 --group-ratio 0.55" "--groups 8 --group-ratio 0.5" "--groups 6 --group-ratio 0.5" "--groups 7 --group-ratio 0.65"; do
  timeout 600 python bench.py --no-cpu-baseline $cfg > gpurun_out/g.json 2> gpurun_out/g.err || tail -3 gpurun_out/g.err
  python - "$cfg" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/g.json").read().strip().splitlines()[-1])
s = d["stages"]
print(sys.argv[1], "| step %.2f e2e %.2f build %.2f kbuild %.2f scan %.2f solve_exp %.3f" % (d["ms_per_step"], d["e2e"]["ms_per_step"], s["scan_build_ms_median"], s["k_build_ms_median"], s["scan_ms_median"], s["solve_exposed_ms_median"]))
PY
done
timeout 600 python bench.py --workload paper_net_energy --reward-sum counts --no-cpu-baseline > gpurun_out/bench_c4_counts.json 2>/dev/null; echo "c4 rc=$?"
timeout 900 python bench.py --workload paper_net_energy --no-cpu-baseline > gpurun_out/bench_c4_seq.json 2>/dev/null; echo "c4seq rc=$?"
timeout 600 python bench.py --workload paper_energy --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null; echo "c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_build|k_vmax" -c 4 -o gpurun_out/prof_r2b -f \
      python tools/profile_build.py paper 1 > gpurun_out/prof_r2b.log 2>&1; echo "ncu rc=$?"
