#!/bin/bash
# k_newton L2 prefetch of the next cell (BTE_NEWTON_PF) on the demo / Fig. 9 / config 2 / config 3 / config 4.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-npf}
: > gpurun_out/ab_${TAG}.jsonl
for R in 1 2; do
for C in 6 10 2 3 4; do
for V in 0 1; do
  ST=400; [ $C = 2 ] && ST=100; [ $C = 3 ] && ST=10; [ $C = 4 ] && ST=5
  L=$(BTE_NEWTON_PF=$V timeout 300 python bench.py --config $C --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'newton_pf': $V, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
cat gpurun_out/ab_${TAG}.jsonl
