# final-lib check: full GPU suite, smoke, ncu --set full of one k_solve_layer (clock-control none)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_solve_layer" -s 50 -c 1 -o gpurun_out/prof_solve -f \
    python tools/profile_build.py paper 1 > gpurun_out/prof_solve.log 2>&1; echo "ncu solve rc=$?"
