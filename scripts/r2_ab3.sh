#!/bin/bash
# A/B: L2 bulk prefetch distance of the sweep's own blocks (BTE_L2PF) and ring depth.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2e}
VARS=${VARS:-"BTE_L2PF=0 BTE_L2PF=2 BTE_L2PF=4 BTE_L2PF=8 BTE_L2PF=4,BTE_SEGS=3 BTE_L2PF=8,BTE_SEGS=3"} CFGS=${CFGS:-"4 3"} TAG=$TAG bash scripts/r2_ab_raster.sh
for V in BTE_L2PF=0 BTE_L2PF=4; do
  env $V timeout 300 python bench.py --config 2 --steps 100 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c2_$V.json 2>&1
done
