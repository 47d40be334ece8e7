#!/bin/bash
# A/B on the headline (config 4): Newton occupancy variants, segment counts, strip width.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2v}
: > gpurun_out/ab_${TAG}.jsonl
for V in BTE_NEWTON_MINB=0 BTE_NEWTON_MINB=2 BTE_NEWTON_MINB=3 BTE_NEWTON_MINB=5 BTE_NEWTON_MINB=6 BTE_SEGS=5 BTE_SEGS=8 BTE_RASTER=20 BTE_RASTER=12; do
  L=$(env $V timeout 300 python bench.py --config 4 --steps 10 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'variant': '$V', 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'bnd_ms': r['device_ms_per_step']['boundary'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done
cat gpurun_out/ab_${TAG}.jsonl
