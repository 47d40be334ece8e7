#!/bin/bash
# Warp-synchronous small-block sweep vs k_sweep on the paper's shapes; parity of the small-block paths.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2z}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "small_3d or config1 or demo or fig9 or inplane or variants or mirror or fixed_point or partial or band or sc_tau" > gpurun_out/pytest_small_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_small_${TAG}.log
: > gpurun_out/ab_${TAG}.jsonl
for C in 6 10 1; do for V in BTE_WARPSWEEP=0 BTE_WARPSWEEP=1 BTE_WARPSWEEP=1,BTE_SEGS=15; do
  ENVS=$(echo $V | tr ',' ' ')
  L=$(env $ENVS timeout 300 python bench.py --config $C --steps 400 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$V', 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'kernel': r['kernel']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done
cat gpurun_out/ab_${TAG}.jsonl; tail -2 gpurun_out/pytest_small_${TAG}.log
