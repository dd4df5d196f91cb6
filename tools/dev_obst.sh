cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "binned or paper_scale or dense_random or desk_parity or smoke_parity or random_env_parity" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
QT_ITERS=5 timeout 300 python tools/quick_time.py paper 2>&1 | tail -1
FM_NO_OBST_BINS=1 QT_ITERS=5 timeout 300 python tools/quick_time.py paper 2>&1 | tail -1
