#!/bin/bash
# Knob sweep on the default launch shapes: segments / strips / stages per workload.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-knobs}
: > gpurun_out/ab_${TAG}.jsonl
run() {  # config steps env...
  local C=$1 ST=$2; shift 2
  L=$(env "$@" timeout 400 python bench.py --config $C --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$*', 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
}
for S in 0 4 6 12 15 24; do run 6 400 BTE_SEGS=$S; done
for S in 0 4 12 20; do run 10 400 BTE_SEGS=$S; done
for S in 0 4 6 12; do run 2 100 BTE_SEGS=$S; done
for S in 2 4; do run 2 100 BTE_STAGES=$S; done
for V in "BTE_SEGS=0" "BTE_SEGS=4" "BTE_RASTER=12" "BTE_RASTER=20" "BTE_SEGS=0"; do run 4 5 $V; done
cat gpurun_out/ab_${TAG}.jsonl
