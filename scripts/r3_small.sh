#!/bin/bash
# Small-block sweep (k_sweep) with running pointers vs the previous build (ablib/libbte_base.so).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-small}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
tail -3 gpurun_out/pytest_${TAG}.log
: > gpurun_out/ab_${TAG}.jsonl
for R in 1 2; do
for C in 6 10 1; do
for V in "BTE_LIB=ablib/libbte_base.so" "BTE_X=new"; do
  L=$(env $V timeout 300 python bench.py --config $C --steps 400 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$V', 'kernel': r['kernel'], 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done; done
cat gpurun_out/ab_${TAG}.jsonl
