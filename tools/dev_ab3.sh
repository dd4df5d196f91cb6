# dev: A/B of k_build launch times (base in-tree lib vs variants), parity of the first variant on the
# obstacle-heavy configs, and an ncu --set full of the variant's lean + obstacle launches at C2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for lib in paper_2109_00857_b200/libflowmdp_b200.so "$@"; do
  FM_LIB_PATH=$lib QT_ITERS=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab.csv \
    python tools/quick_time.py ${W:-paper} > /dev/null 2>&1
  echo "== $lib"; python tools/kernel_times.py gpurun_out/ab.csv 2 2>&1 | grep -E "k_build|k_vmax"
done
V=$1
if [ -n "$V" ]; then
  FM_LIB_PATH=$V timeout 1200 python -m pytest tests/test_gpu_bench_configs.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo "variant tests rc=$?"; tail -2 gpurun_out/ab_tests.log
  FM_LIB_PATH=$V timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_build" -s 0 -c 30 -o gpurun_out/prof_v -f \
      python tools/profile_build.py paper 1 > gpurun_out/prof_v.log 2>&1; echo "ncu rc=$?"
fi
