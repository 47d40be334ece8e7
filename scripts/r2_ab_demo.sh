#!/bin/bash
# A/B: segment count for the paper's small-block shapes (demo, Fig. 9) and config 1.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2n}
: > gpurun_out/ab_${TAG}.jsonl
for C in 6 10; do for V in BTE_SEGS=0 BTE_SEGS=4 BTE_SEGS=15 BTE_SEGS=24 BTE_SEGS=30 BTE_SEGS=60; do
  L=$(env $V timeout 300 python bench.py --config $C --steps 400 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$V', 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'newton_ms': r['device_ms_per_step']['newton']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done
cat gpurun_out/ab_${TAG}.jsonl
