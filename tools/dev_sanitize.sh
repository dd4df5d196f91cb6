# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py -> gpurun_out/sanitizer/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
python tools/sanitize_cases.py > gpurun_out/sanitizer/plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer/$tool.log
done
