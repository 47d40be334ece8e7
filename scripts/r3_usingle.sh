#!/bin/bash
# Unstructured sweep on triangles: one neighbour buffer + 2 CTAs/SM (BTE_USINGLE=1) vs the default.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-usingle}
BTE_USINGLE=1 timeout 600 python -m pytest tests/test_gpu_umesh.py -m gpu -x -q -rf 2>&1 | tail -3
: > gpurun_out/ab_${TAG}.jsonl
for R in 1 2; do
for V in 0 1; do
  L=$(BTE_USINGLE=$V timeout 300 python bench.py --config 7 --steps 40 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': 7, 'usingle': $V, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done
cat gpurun_out/ab_${TAG}.jsonl
