#!/bin/bash
# ncu --set full of the unstructured sweep (u2, u3), pipelined and plain variants.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r03}
for CFG in ${CFGS:-7 8}; do
  for V in ${VARS:-tma plain}; do
    R=gpurun_out/prof_usweep_${V}_${TAG}_c${CFG}
    if [ $V = plain ]; then export BTE_SWEEP=plain; else unset BTE_SWEEP; fi
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_usweep -s 2 -c 1 \
      -o $R -f python scripts/prof_step.py --config $CFG --warmup 2 --steps 1 > $R.log 2>&1
    python scripts/ncu_summary.py rep $R.ncu-rep --workload c$CFG > $R.json
    if [ "$V$CFG" != "tma7" ]; then rm -f $R.ncu-rep; fi
  done
done
unset BTE_SWEEP
ls -la gpurun_out/*.ncu-rep
