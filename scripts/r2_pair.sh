#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2ab}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "small_3d or config1 or demo or fig9 or inplane or mirror or fixed_point or partial or band" > gpurun_out/pytest_pair_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pair_${TAG}.log
: > gpurun_out/ab_${TAG}.jsonl
for C in 6 10 1; do for V in BTE_PAIR=0 BTE_PAIR=1; do
  L=$(env $V timeout 300 python bench.py --config $C --steps 400 --repeats 3 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$V', 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done
cat gpurun_out/ab_${TAG}.jsonl; tail -2 gpurun_out/pytest_pair_${TAG}.log
