cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "reward_sum or binned or smoke_parity or desk_parity or deterministic" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
for RS in counts sequential; do
timeout 600 python bench.py --workload paper_net_energy --reward-sum $RS --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c4_$RS.json 2> gpurun_out/bench_c4_$RS.err; echo "c4 $RS rc=$?"; tail -2 gpurun_out/bench_c4_$RS.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_c4_$RS.json').read().strip().splitlines()[-1]); print('$RS ms', round(d['ms_per_step'],2), 'e2e', round(d['e2e']['ms_per_step'],2), {k: round(v,2) if isinstance(v,float) else v for k,v in d['stages'].items() if k!='strips'}, d['roofline']['frac'])"
done
