# dev: N=2 gloo validation + C3/C4 bench lines (no CPU baseline)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --gpus 2 --dist-backend gloo --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; echo "gloo2 rc=$?"; tail -2 gpurun_out/bench_gloo2.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_gloo2.json').read().strip().splitlines()[-1]); print('gloo2', d['n_gpus'], d['stages'])"
for W in paper_energy paper_net_energy; do
timeout 600 python bench.py --workload $W --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err; echo "$W rc=$?"; tail -2 gpurun_out/bench_$W.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_$W.json').read().strip().splitlines()[-1]); print('$W ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), {k: round(v,2) if isinstance(v,float) else v for k,v in d['stages'].items() if k!='strips'})"
done
