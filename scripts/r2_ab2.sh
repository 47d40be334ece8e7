#!/bin/bash
# GPU tests of the implicit step + A/B of the reworked TMA sweep (compile-time
# ring depth, 72-register bound) on configs 4/3/2 with segment variants.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2d}
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "implicit" > gpurun_out/pytest_imp_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_imp_${TAG}.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
VARS="BTE_RASTER=16 BTE_RASTER=0 BTE_RASTER=16,BTE_SEGS=3 BTE_RASTER=24,BTE_SEGS=4" CFGS="4 3" TAG=$TAG bash scripts/r2_ab_raster.sh
for A in "--config 2 --steps 100"; do
  timeout 300 python bench.py $A --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c2.json 2>&1
done
tail -3 gpurun_out/pytest_imp_${TAG}.log; tail -3 gpurun_out/pytest_gpu_${TAG}.log
