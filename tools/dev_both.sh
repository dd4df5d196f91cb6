cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "binned or paper_scale or dense_random or desk_parity or smoke_parity or random_env_parity" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
QT_ITERS=5 timeout 300 python tools/quick_time.py paper 2>&1 | tail -1
FM_NO_OBST_BINS=1 QT_ITERS=5 timeout 300 python tools/quick_time.py paper 2>&1 | tail -1
# dev: per-kernel times of a few builds (ncu launch list) + path statistics
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
W=${1:-paper}
QT_ITERS=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qt_launches.csv \
    python tools/quick_time.py $W > /dev/null 2>&1
python tools/kernel_times.py gpurun_out/qt_launches.csv 2>&1 | head -20
[ -f paper_2109_00857_b200/libflowmdp_stats.so ] && FM_LIB_PATH=paper_2109_00857_b200/libflowmdp_stats.so timeout 300 python tools/stats_probe.py $W 2>&1 | tail -1
[ -f paper_2109_00857_b200/libflowmdp_stats.so ] && FM_NO_OBST_BINS=1 FM_LIB_PATH=paper_2109_00857_b200/libflowmdp_stats.so timeout 300 python tools/stats_probe.py $W 2>&1 | tail -1
