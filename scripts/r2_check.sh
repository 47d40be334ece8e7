#!/bin/bash
# Full GPU suite + graph A/B on the launch-sensitive shapes + default bench line.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2h}
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
for C in 6 1 10 2; do for G in 0 1; do
  BTE_GRAPH=$G timeout 300 python bench.py --config $C --steps 200 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c${C}_g$G.json 2>&1
done; done
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -3 gpurun_out/pytest_gpu_${TAG}.log
