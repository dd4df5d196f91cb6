cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; tail -3 gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','stages','clocks','gpu_launches')}); print('e2e', d['e2e']['ms_per_step'], 'dropin', d['e2e_dropin']['ms_per_step'], d['roofline'], d['issue_roofline'])"
timeout 600 python bench.py --gpus 3 --dist-backend gloo --steps 2 --warmup 1 --workload desk > gpurun_out/bench_gloo3.json 2> gpurun_out/bench_gloo3.err; echo gloo3 rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_gloo3.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('n_gpus','value','ms_per_step','stages')})"
