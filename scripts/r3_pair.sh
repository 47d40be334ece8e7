#!/bin/bash
# Two x-adjacent columns per CTA (BTE_PAIR=1): parity subset, then A/B vs k_sweep_tma on configs 3/4 (+ ncu DRAM bytes).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-pair}
BTE_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -rf -k "config3 or config4 or config5 or rotation or all_bc or random_problems or degenerate or slab or temperature_only" > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_${TAG}.log
tail -4 gpurun_out/pytest_${TAG}.log
BTE_PAIR=1 timeout 120 python __graft_entry__.py --smoke 2>&1 | head -1
: > gpurun_out/ab_${TAG}.jsonl
for R in 1 2; do
for C in 3 4; do
for V in 0 1; do
  L=$(BTE_PAIR=$V timeout 400 python bench.py --config $C --steps 10 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'pair': $V, 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done; done
cat gpurun_out/ab_${TAG}.jsonl
for V in 0 1; do
BTE_PAIR=$V timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_sweep -s 3 -c 1 --csv \
  python scripts/prof_step.py --config 3 --warmup 3 --steps 1 2>/dev/null | grep -E 'dram__bytes|duration|hit_rate|sm__throughput' | awk -F'","' -v v=$V '{print "pair=" v, $5, $(NF-2), $NF}'
done
