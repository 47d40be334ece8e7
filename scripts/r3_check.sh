#!/bin/bash
# Smoke, full GPU suite, default bench line (state check at session start).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-s3}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=15 > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
tail -3 gpurun_out/pytest_gpu_${TAG}.log; cat gpurun_out/smoke_${TAG}.log; cut -c1-400 gpurun_out/bench_${TAG}.json
