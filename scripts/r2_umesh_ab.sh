#!/bin/bash
# Unstructured sweep variants: ring depth / chunk size on u2 and u3; the hexahedral line (config 11).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2x}
: > gpurun_out/ab_${TAG}.jsonl
for C in 7 8; do for V in BTE_STAGES=0 BTE_STAGES=4 BTE_SEGS=32 BTE_SEGS=128 BTE_THREADS=500 BTE_THREADS=1000; do
  L=$(env $V timeout 300 python bench.py --config $C --steps 20 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$V', 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done
timeout 600 python bench.py --config 11 --steps 5 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c11.json 2>&1
cat gpurun_out/ab_${TAG}.jsonl; tail -c 400 gpurun_out/bench_${TAG}_c11.json
