#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for cfg in ${CFGS:-2 6}; do
  echo "== config $cfg"
  BTE_NEWTON_STATS=1 timeout 300 python scripts/prof_step.py --config $cfg --warmup ${W:-300} --steps 10 2>&1 | grep -E "stats|done" | tail -3
done
