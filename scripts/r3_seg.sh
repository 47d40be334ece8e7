#!/bin/bash
# 3-D sweep column order: segments along the march axis x strip width; bench time + ncu DRAM bytes per launch.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-seg}
: > gpurun_out/ab_${TAG}.jsonl
for C in 4 3; do
for V in "BTE_SEGS=0" "BTE_SEGS=1" "BTE_SEGS=2" "BTE_SEGS=3" "BTE_SEGS=1 BTE_RASTER=24" "BTE_SEGS=1 BTE_RASTER=32" "BTE_SEGS=2 BTE_RASTER=32" "BTE_SEGS=1 BTE_RASTER=10"; do
  L=$(env $V timeout 300 python bench.py --config $C --steps 10 --repeats 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  SK=3; [ $C = 4 ] && SK=9
  env $V timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_sweep -s $SK -c 1 --csv \
      python scripts/prof_step.py --config $C --warmup 3 --steps 1 > gpurun_out/ncu_${TAG}.csv 2>/dev/null
  python - "$L" "$C" "$V" gpurun_out/ncu_${TAG}.csv >> gpurun_out/ab_${TAG}.jsonl <<'PY'
import json, sys, csv, io
d = json.loads(sys.argv[1]); r = d['roofline']; C = int(sys.argv[2])
txt = open(sys.argv[4]).read(); i = txt.find('"ID"'); m = {}
if i >= 0:
    for row in csv.DictReader(io.StringIO(txt[i:])):
        m[row['Metric Name']] = float(row['Metric Value'].replace(',', '')) * {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1, 'ms': 1e-3, 'msecond': 1e-3, 'us': 1e-6, 'usecond': 1e-6, 'ns': 1e-9, 'nsecond': 1e-9, '%': 1}.get(row['Metric Unit'], 1)
dof = {4: 2e9, 3: 4194304000}[C]
out = {'config': C, 'variant': sys.argv[3], 'ms_per_step': d['ms_per_step'], 'sweep_ms': r['kernel_ms_avg'], 'frac': r['frac'], 'mhz': d['clocks']['sm_mhz']}
if 'dram__bytes_read.sum' in m:
    out['ncu_ms'] = m['gpu__time_duration.sum'] * 1e3
    out['ncu_B_per_dof'] = (m['dram__bytes_read.sum'] + m['dram__bytes_write.sum']) / dof
    out['ncu_frac'] = 16 * dof / m['gpu__time_duration.sum'] / 6.5398e12
    out['l2_hit'] = m.get('lts__t_sector_hit_rate.pct')
print(json.dumps(out))
PY
done; done
cat gpurun_out/ab_${TAG}.jsonl
