#!/bin/bash
# k_newton residency (BTE_NEWTON_MINB blocks of 8 warps per SM) on the small shapes (wave quantisation) and config 3.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-minb}
: > gpurun_out/ab_${TAG}.jsonl
for C in 6 10 2 1 3; do
for V in 4 5 6 3; do
  ST=400; [ $C = 2 ] && ST=100; [ $C = 3 ] && ST=10
  L=$(BTE_NEWTON_MINB=$V timeout 300 python bench.py --config $C --steps $ST --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'minb': $V, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done
cat gpurun_out/ab_${TAG}.jsonl
