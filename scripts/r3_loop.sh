#!/bin/bash
# Loopback multi-rank tests on one GPU; Newton with the band-index table in shared memory vs ablib/libbte_base.so.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-loop}
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q -rf > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
tail -5 gpurun_out/pytest_${TAG}.log
: > gpurun_out/ab_${TAG}.jsonl
for R in 1 2; do
for C in 6 10 2 3; do
for V in "BTE_LIB=ablib/libbte_base.so" "BTE_X=sib"; do
  ST=400; [ $C = 2 ] && ST=100; [ $C = 3 ] && ST=10
  L=$(env $V timeout 300 python bench.py --config $C --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$V', 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done; done
cat gpurun_out/ab_${TAG}.jsonl
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -5
