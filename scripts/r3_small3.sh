#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "demo or small or fig9 or config1 or inplane or degenerate" 2>&1 | tail -1
: > gpurun_out/lines_small3.jsonl
for R in 1 2; do for A in "--config 6 --steps 400" "--config 10 --steps 400" "--config 1 --steps 400"; do
  timeout 600 python bench.py $A --warmup 3 --repeats 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> gpurun_out/lines_small3.jsonl
done; done
python -c "
import json
for l in open('gpurun_out/lines_small3.jsonl'):
    d=json.loads(l); r=d['roofline']; print(d['config']['workload'], round(d['ms_per_step'],4), round(r['frac'],3), round(r['kernel_ms_avg'],5), round(r['device_ms_per_step']['newton'],4))"
