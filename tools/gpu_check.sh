#!/bin/bash
# GPU-box check used during development: GPU tests, the bench (N=1), the
# N=2 path validated with gloo on one GPU, a short reference arm.  Outputs
# under gpurun_out/.  Usage: tools/gpu_check.sh [pytest -k expression]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -1 gpurun_out/smoke.log
K=${1:+-k "$1"}
timeout 1500 python -m pytest tests -m gpu -x -q $K > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench.json
timeout 600 python bench.py --gpus 2 --dist-backend gloo --steps 2 --warmup 1 --no-cpu-baseline \
    > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; echo "gloo2 rc=$?"
tail -c 600 gpurun_out/bench_gloo2.json; tail -5 gpurun_out/bench_gloo2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref rc=$?"
tail -c 1500 gpurun_out/ref.json
