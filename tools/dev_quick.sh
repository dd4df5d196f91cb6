# dev: binned-path parity subset + C2 build timing (+ per-kernel launch list)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${PT_K:-binned or paper_scale or dense_random or desk_parity or smoke_parity or random_env_parity}" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
QT_ITERS=6 timeout 300 python tools/quick_time.py ${1:-paper} 2>&1 | tail -1
QT_ITERS=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qt_launches.csv \
    python tools/quick_time.py ${1:-paper} > /dev/null 2>&1
python tools/kernel_times.py gpurun_out/qt_launches.csv 2 2>&1 | grep -v "at::\|k_mask\|k_prob\|k_gate\|maxabs"
