#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/ab_imporder.jsonl
BTE_IMP_ORDER=1 timeout 600 python -m pytest tests -m gpu -x -q -k "implicit" 2>&1 | tail -1
BTE_IMP_ORDER=2 timeout 600 python -m pytest tests -m gpu -x -q -k "implicit" 2>&1 | tail -1
for R in 1 2; do for C in 3 2; do for V in 0 1 2; do
  ST=2; [ $C = 2 ] && ST=20
  L=$(BTE_IMP_ORDER=$V timeout 400 python bench.py --config $C --implicit 4 --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'order': $V, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_imporder.jsonl
done; done; done
cat gpurun_out/ab_imporder.jsonl
