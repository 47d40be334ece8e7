#!/bin/bash
# ncu evidence: launch list of a short bench run + one --set full capture of the sweep and the Newton.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${CFG:-2}
TAG=${TAG:-r01}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_c${CFG}.csv \
  python scripts/prof_step.py --config $CFG --warmup 3 --steps 3 > gpurun_out/launches_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 \
  -o gpurun_out/prof_sweep_${TAG}_c${CFG} -f python scripts/prof_step.py --config $CFG --warmup 3 --steps 1 > gpurun_out/prof_sweep_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_newton -s 3 -c 1 \
  -o gpurun_out/prof_newton_${TAG}_c${CFG} -f python scripts/prof_step.py --config $CFG --warmup 3 --steps 1 > gpurun_out/prof_newton_${TAG}.log 2>&1
ls -la gpurun_out
