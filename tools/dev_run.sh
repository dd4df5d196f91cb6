cd $GRAFT_REPO_ROOT
timeout 300 python tools/quick_time.py paper 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p2.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/p2.log
