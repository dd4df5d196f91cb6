# dev: halo-hook ABI test, sharded tests, net-energy count-reward tests + C4 line (in-tree lib)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q -m gpu > gpurun_out/halo_tests.log 2>&1; echo "sharded/halo tests rc=$?"; tail -1 gpurun_out/halo_tests.log
bash tools/dev_netr.sh paper_2109_00857_b200/libflowmdp_b200.so
