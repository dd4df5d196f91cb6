# dev: C2 build timing of the in-tree library and of variants (FM_LIB_PATH)
cd $GRAFT_REPO_ROOT
for lib in paper_2109_00857_b200/libflowmdp_b200.so "$@"; do
  echo "== $lib"; FM_LIB_PATH=$lib QT_ITERS=6 timeout 300 python tools/quick_time.py ${W:-paper} 2>&1 | tail -1
done
