#!/bin/bash
# k_sweep (small blocks): L2 prefetch distance BTE_PF on the paper's demo / Fig. 9 shapes and config 1.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-pf}
: > gpurun_out/ab_${TAG}.jsonl
for R in 1 2; do
for C in 6 10 1; do
for V in 0 1 2 4; do
  L=$(BTE_PF=$V timeout 300 python bench.py --config $C --steps 400 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'pf': $V, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done; done
BTE_PF=2 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "demo or small or fig9 or config1" 2>&1 | tail -1
cat gpurun_out/ab_${TAG}.jsonl
