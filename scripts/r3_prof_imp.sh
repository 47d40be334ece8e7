#!/bin/bash
# ncu --set full (+ source) of the implicit wavefront sweep on config 3 (4 iterations/step, 8x dt).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R=gpurun_out/prof_imp_c3
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_sweep_imp -s 2 -c 1 -o $R -f \
  python bench.py --config 3 --implicit 4 --steps 1 --warmup 3 --repeats 1 --no-cpu-baseline --no-e2e > $R.log 2>&1
python scripts/ncu_summary.py rep $R.ncu-rep --workload "config3_3d_si_64^3x400x40 implicit" --dof 4194304000 > $R.json
ncu -i $R.ncu-rep --page source --csv > $R.src.csv 2>/dev/null
ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
rm -f $R.ncu-rep
tail -3 $R.log; du -sh gpurun_out
