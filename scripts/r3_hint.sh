#!/bin/bash
# mbarrier try_wait with a suspend-time hint vs without (ablib/libbte_base.so): 3-D / 2-D TMA sweeps, unstructured.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-hint}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
: > gpurun_out/ab_${TAG}.jsonl
for R in 1 2; do
for C in 3 4 2 7; do
for V in "BTE_LIB=ablib/libbte_base.so" "BTE_X=hint"; do
  ST=10; [ $C = 2 ] && ST=100; [ $C = 7 ] && ST=40
  L=$(env $V timeout 300 python bench.py --config $C --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$V', 'kernel': r['kernel'], 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done; done
cat gpurun_out/ab_${TAG}.jsonl
