#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2w}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "rotation or config4 or partial or semi" > gpurun_out/pytest_ov_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_ov_${TAG}.log
timeout 300 python bench.py --config 4 --steps 20 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c4.json 2>&1
tail -2 gpurun_out/pytest_ov_${TAG}.log
