#!/bin/bash
# k_sweep_pc (producer/consumer chunk ring): parity subset, then A/B against k_sweep_tma.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-pc1}
timeout 120 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
cat gpurun_out/smoke_${TAG}.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config3 or config2 or config4 or variants or slot_rotation or all_bc or random_problems" > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
tail -5 gpurun_out/pytest_${TAG}.log
: > gpurun_out/ab_${TAG}.jsonl
for C in 3 2 4; do
for V in BTE_SWEEP=tma BTE_SWEEP=pc BTE_STAGES=4 BTE_STAGES=6 BTE_STAGES=8; do
  ST=10; [ $C = 2 ] && ST=100
  L=$(env $V timeout 300 python bench.py --config $C --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$V', 'kernel': r['kernel'], 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done
cat gpurun_out/ab_${TAG}.jsonl
