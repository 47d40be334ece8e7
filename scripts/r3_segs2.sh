#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/ab_segs2.jsonl
for R in 1 2; do for C in 10 1 6; do
  L=$(timeout 400 python bench.py --config $C --steps 400 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton']}))" "$L" >> gpurun_out/ab_segs2.jsonl
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fig9 or config1 or demo or small" 2>&1 | tail -1
cat gpurun_out/ab_segs2.jsonl
