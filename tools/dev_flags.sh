# dev: launch list of quick_time under FM_DEV_FLAGS values (timing A/B only: results may be wrong)
cd $GRAFT_REPO_ROOT
for f in ${FLAGS_LIST:-0 1}; do
FM_DEV_FLAGS=$f QT_ITERS=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qt_f$f.csv \
    python tools/quick_time.py ${W:-paper} > /dev/null 2>&1
echo "== FM_DEV_FLAGS=$f"; python tools/kernel_times.py gpurun_out/qt_f$f.csv 2 2>&1 | grep "k_build\|k_vmax"
done
