# dev: k_vmax step variants (scan stage) and upload slab counts (e2e), one bench line each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() {
  timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/g.json 2> gpurun_out/g.err || tail -3 gpurun_out/g.err
  python - "$FM_LIB_PATH $*" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/g.json").read().strip().splitlines()[-1]); s = d["stages"]
print(sys.argv[1], "| step %.2f e2e %.2f kbuild %.2f scan %.2f" % (d["ms_per_step"], d["e2e"]["ms_per_step"], s["k_build_ms_median"], s["scan_ms_median"]))
PY
}
run
FM_LIB_PATH=abl/vs8.so run
FM_LIB_PATH=abl/vs2.so run
run --upload-slabs 16
run --upload-slabs 4
run
