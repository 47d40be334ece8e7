#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2aa}
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
for C in 1 6 10; do
  timeout 300 python bench.py --config $C --steps 400 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c$C.json 2>/dev/null
done
tail -2 gpurun_out/pytest_gpu_${TAG}.log
