#!/bin/bash
# Implicit sweep with L2 policies (BTE_IMP_L2=1: own I^n evict-first, I^{k+1} evict-last) vs without.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-impl2}
timeout 900 python -m pytest tests -m gpu -x -q -k "implicit" 2>&1 | tail -2
: > gpurun_out/ab_${TAG}.jsonl
for R in 1 2; do
for C in 3 2; do
for V in 0 1; do
  ST=2; [ $C = 2 ] && ST=20
  L=$(BTE_IMP_L2=$V timeout 400 python bench.py --config $C --implicit 4 --steps $ST --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'imp_l2': $V, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done; done
for V in 0 1; do
BTE_IMP_L2=$V timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_sweep_imp -s 2 -c 1 --csv \
  python bench.py --config 3 --implicit 4 --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E 'dram__bytes|duration|hit_rate' | sed "s/^/imp_l2=$V /"
done
cat gpurun_out/ab_${TAG}.jsonl
