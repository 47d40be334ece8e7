#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2y}
timeout 1200 python -m pytest tests/test_gpu_umesh.py -q -x > gpurun_out/pytest_umesh_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_umesh_${TAG}.log
timeout 600 python bench.py --config 11 --steps 10 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c11.json 2>&1
timeout 600 python bench.py --config 8 --steps 10 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c8.json 2>&1
tail -2 gpurun_out/pytest_umesh_${TAG}.log
