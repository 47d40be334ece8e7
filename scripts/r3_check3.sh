#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-check3}
timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
tail -3 gpurun_out/smoke_${TAG}.log
: > gpurun_out/lines_${TAG}.jsonl
for A in "--config 7 --steps 40" "--config 9 --steps 40" "--config 8 --steps 10"; do
  timeout 600 python bench.py $A --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> gpurun_out/lines_${TAG}.jsonl
done
python -c "
import json
for l in open('gpurun_out/lines_${TAG}.jsonl'):
    d=json.loads(l); r=d['roofline']; print(d['config']['workload'], round(d['ms_per_step'],4), '%.3e'%d['value'], round(r['frac'],3), round(r['kernel_ms_avg'],4))"
