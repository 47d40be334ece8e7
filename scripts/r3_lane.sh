#!/bin/bash
# Lane-per-cell Newton: parity tests, full GPU suite, A/B against the warp-per-cell k_newton (BTE_NEWTON_LANE=0).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-lane}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -rf -k "lane" > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
tail -4 gpurun_out/pytest_${TAG}.log
: > gpurun_out/ab_${TAG}.jsonl
for C in 3 4 8 5; do
for V in 0 1; do
  ST=10; [ $C = 4 ] && ST=5
  L=$(BTE_NEWTON_LANE=$V timeout 400 python bench.py --config $C --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'lane': $V, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done
cat gpurun_out/ab_${TAG}.jsonl
timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
tail -4 gpurun_out/pytest_gpu_${TAG}.log
