#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2j}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k implicit > gpurun_out/pytest_imp_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_imp_${TAG}.log
for V in "BTE_THREADS=0"; do
  env $V timeout 300 python bench.py --config 3 --implicit 4 --steps 2 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$V.json 2>&1
done
tail -2 gpurun_out/pytest_imp_${TAG}.log
