# dev: the N>1 bench path on one GPU over gloo (validation, never a bench number)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/n2.json 2> gpurun_out/n2.err; echo "n2 rc=$?"; tail -3 gpurun_out/n2.err
python -c "import json; d=json.loads(open('gpurun_out/n2.json').read().strip().splitlines()[-1]); print({k: d.get(k) for k in ('n_gpus','ms_per_step','value')}, d['config'].get('parallelism'), d['stages'].get('strips'))"
