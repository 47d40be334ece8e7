#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for CFG in ${CFGS:-2 6}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_newton -s 20 -c 1 \
  -o gpurun_out/prof_newton_${TAG}_c${CFG} -f python scripts/prof_step.py --config $CFG --warmup 20 --steps 1 > gpurun_out/prof_newton_${TAG}_c${CFG}.log 2>&1
done
ls gpurun_out
