# dev: ncu --set full of one k_build PART-2 launch (obstacle tasks)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k k_build -s ${SKIP:-1} -c 1 -o gpurun_out/prof_p${SKIP:-1} -f \
    python tools/profile_build.py ${1:-paper} 1 > gpurun_out/prof_p2.log 2>&1
tail -3 gpurun_out/prof_p2.log
