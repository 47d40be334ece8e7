#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/ab_lpc.jsonl
BTE_NEWTON_LPC=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "demo or config2 or config3 or set_state or fixed_point or newton or solve" 2>&1 | tail -1
for R in 1 2; do for C in 6 10 2 3 4; do for V in 0 1; do
  ST=400; [ $C = 2 ] && ST=100; [ $C = 3 ] && ST=10; [ $C = 4 ] && ST=5
  L=$(BTE_NEWTON_LPC=$V timeout 400 python bench.py --config $C --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'lpc': $V, 'ms_per_step': d['ms_per_step'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_lpc.jsonl
done; done; done
cat gpurun_out/ab_lpc.jsonl
