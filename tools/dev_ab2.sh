# dev: per-kernel times (launch list) of quick_time for the in-tree lib and variants
cd $GRAFT_REPO_ROOT
for lib in paper_2109_00857_b200/libflowmdp_b200.so "$@"; do
  FM_LIB_PATH=$lib QT_ITERS=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab.csv \
    python tools/quick_time.py ${W:-paper} > /dev/null 2>&1
  echo "== $lib"; python tools/kernel_times.py gpurun_out/ab.csv 2 2>&1 | grep "k_build"
done
