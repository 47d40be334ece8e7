#!/bin/bash
# A/B: 3-D y-upwind by direct L2 loads (BTE_YDIRECT) vs staged; graph replay on small shapes.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2g}
VARS=${VARS:-"BTE_YDIRECT=0 BTE_YDIRECT=1 BTE_YDIRECT=1,BTE_SEGS=3 BTE_YDIRECT=1,BTE_RASTER=32 BTE_YDIRECT=1,BTE_STAGES=2"} CFGS=${CFGS:-"4 3"} TAG=$TAG bash scripts/r2_ab_raster.sh
for C in 6 1 10; do for G in 0 1; do
  BTE_GRAPH=$G timeout 300 python bench.py --config $C --steps 200 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c${C}_g$G.json 2>&1
done; done
BTE_YDIRECT=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config3 or config4 or config5 or small_3d or slab or rotation" > gpurun_out/pytest_yd_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_yd_${TAG}.log
timeout 900 python -m pytest tests -q -x -m gpu -k "umesh or graph or step_splitting or newton_failure or determinism" > gpurun_out/pytest_misc_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_misc_${TAG}.log
