#!/bin/bash
# A/B of sweep variants (env knobs of libbte) on the bench workload; no e2e / cpu legs.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
OUT=gpurun_out/ab_${TAG:-x}.txt
: > $OUT
for v in ${VARIANTS:-"BTE_SWEEP=plain" "BTE_STAGES=2" "BTE_STAGES=3" "BTE_STAGES=4"}; do
  for cfg in ${CFGS:-2}; do
    line=$(env ${v//,/ } timeout 300 python bench.py --config $cfg --steps ${STEPS:-200} --warmup ${WARM:-5} --no-e2e --no-cpu-baseline 2>>gpurun_out/ab_err.txt)
    echo "$v cfg=$cfg $(echo "$line" | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; dm=r["device_ms_per_step"]; c=d.get("clocks") or {}; print("value=%.4g ms/step=%.4f sweep_ms/step=%.4f newton_ms/step=%.4f frac=%.3f sm_mhz=%s reasons=%s" % (d["value"], d["ms_per_step"], dm["sweep"], dm["newton"], r["frac"], c.get("sm_mhz"), ",".join(c.get("reasons") or [])))')" >> $OUT
  done
done
cat $OUT
