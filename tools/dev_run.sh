cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
timeout 300 python tools/sanitize_cases.py > gpurun_out/sanitizer/plain.log 2>&1; echo plain rc=$?; tail -8 gpurun_out/sanitizer/plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitizer/$tool.log 2>&1; echo $tool rc=$?; tail -4 gpurun_out/sanitizer/$tool.log
done
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','stages','clocks')}); print(d['e2e']['ms_per_step'], d['roofline']['frac'], d['cpu_baseline']['value'])"
