#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2i}
timeout 1200 python -m pytest tests/test_gpu_umesh.py -q -x > gpurun_out/pytest_umesh_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_umesh_${TAG}.log
for IT in 4 8; do
  timeout 600 python bench.py --config 3 --implicit $IT --steps 3 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_imp$IT.json 2>&1
done
timeout 600 python bench.py --config 2 --implicit 4 --steps 10 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c2imp4.json 2>&1
tail -3 gpurun_out/pytest_umesh_${TAG}.log
