#!/bin/bash
# Single-buffer two-CTA unstructured sweep on triangles and tetrahedra/quadrilaterals (BTE_USINGLE=1 default) vs 0.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-usingle2}
timeout 900 python -m pytest tests/test_gpu_umesh.py tests/test_gpu_loopback.py -m gpu -x -q -rf 2>&1 | tail -3
: > gpurun_out/ab_${TAG}.jsonl
for R in 1 2; do for C in 8 9 7; do for VV in "BTE_LIB=ablib/libbte_base.so" "BTE_X=early"; do
  ST=40; [ $C = 8 ] && ST=10
  L=$(env $VV timeout 400 python bench.py --config $C --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$VV', 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done; done
cat gpurun_out/ab_${TAG}.jsonl
