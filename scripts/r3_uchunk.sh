#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/ab_uchunk.jsonl
for R in 1 2; do for C in 8 7; do for Q in 0 32 128 256; do
  ST=10; [ $C = 7 ] && ST=40
  L=$(BTE_SEGS=$Q timeout 400 python bench.py --config $C --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'chunk': $Q, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac']}))" "$L" >> gpurun_out/ab_uchunk.jsonl
done; done; done
cat gpurun_out/ab_uchunk.jsonl
