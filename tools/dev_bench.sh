# dev: bench at N=1 with 1 and 5 slab groups (no CPU baseline)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for G in ${GROUPS_LIST:-1 5}; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --groups $G $EXTRA > gpurun_out/bench_g$G.json 2> gpurun_out/bench_g$G.err; echo "bench G=$G rc=$?"; tail -2 gpurun_out/bench_g$G.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_g$G.json').read().strip().splitlines()[-1])
print('ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), 'd2h', d['e2e']['d2h_bytes_per_step'], {k: round(v,2) if isinstance(v,float) else v for k,v in d['stages'].items() if k!='strips'}, 'frac', round(d['roofline']['frac'],3), 'launches', d['gpu_launches'])"
done
