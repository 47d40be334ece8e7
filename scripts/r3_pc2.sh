#!/bin/bash
# k_sweep_pc chunk sizes (BTE_PC_KC = direction groups per chunk) vs k_sweep_tma; ncu of pc on config 3.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-pc2}
for K in 2 5; do
  BTE_PC_KC=$K timeout 120 python __graft_entry__.py --smoke 2>&1 | head -1 >> gpurun_out/smoke_${TAG}.log
  BTE_PC_KC=$K timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config3_reduced or config2_reduced or all_bc" 2>&1 | tail -1 >> gpurun_out/smoke_${TAG}.log
done
cat gpurun_out/smoke_${TAG}.log
: > gpurun_out/ab_${TAG}.jsonl
for C in 3 4; do
for V in BTE_SWEEP=tma BTE_PC_KC=1 BTE_PC_KC=2 BTE_PC_KC=5; do
  L=$(env $V timeout 300 python bench.py --config $C --steps 10 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[1]); r=d['roofline']; print(json.dumps({'config': $C, 'variant': '$V', 'kernel': r['kernel'], 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'newton_ms': r['device_ms_per_step']['newton'], 'mhz': d['clocks']['sm_mhz']}))" "$L" >> gpurun_out/ab_${TAG}.jsonl
done; done
cat gpurun_out/ab_${TAG}.jsonl
for K in 1 5; do
R=gpurun_out/prof_pc${K}_c3
BTE_PC_KC=$K timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 \
    -o $R -f python scripts/prof_step.py --config 3 --warmup 3 --steps 1 > $R.log 2>&1
python scripts/ncu_summary.py rep $R.ncu-rep --workload "config3_3d_si_64^3x400x40" --dof 4194304000 > $R.json; ncu -i $R.ncu-rep --page source --csv > $R.src.csv 2>/dev/null; rm -f $R.ncu-rep
done
du -sh gpurun_out
