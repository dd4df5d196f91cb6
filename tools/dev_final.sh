# full bench (N=1, default) + reference arm + evidence
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
timeout 600 python bench.py --workload paper_net_energy --reward-sum counts --no-cpu-baseline > gpurun_out/bench_c4_counts.json 2>/dev/null
timeout 600 python bench.py --workload paper_energy --no-cpu-baseline > gpurun_out/bench_c3.json 2>/dev/null
bash tools/profile_r02b.sh
