#!/bin/bash
# A/B: ring depth vs CTAs per SM (BTE_STAGES / BTE_SMEM_KB) on configs 4 and 3.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2f}
VARS=${VARS:-"BTE_STAGES=2 BTE_STAGES=3 BTE_STAGES=4 BTE_STAGES=3,BTE_SEGS=3 BTE_STAGES=4,BTE_SEGS=3 BTE_STAGES=4,BTE_RASTER=32,BTE_SEGS=3"} CFGS=${CFGS:-"4 3"} TAG=$TAG bash scripts/r2_ab_raster.sh
