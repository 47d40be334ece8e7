#!/bin/bash
# A/B of the unstructured sweep variants on u2 / u3 (device ms per step).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
OUT=gpurun_out/umesh_ab.txt
: > $OUT
timeout 600 python -m pytest tests/test_gpu_umesh.py -q -x > gpurun_out/pytest_umesh.log 2>&1; echo "pytest exit $?" >> $OUT
for CFG in ${CFGS:-7 8}; do
  for V in ${VARIANTS:-"BTE_SWEEP=plain" "X=0" "BTE_SEGS=16" "BTE_SEGS=64" "BTE_SEGS=128" "BTE_STAGES=4" "BTE_THREADS=500"}; do
    r=$(env $V timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('%.3f ms sweep %.3f frac %.3f' % (d['ms_per_step'], r['kernel_ms_avg'], r['frac']))")
    echo "cfg $CFG $V: $r" >> $OUT
  done
done
cat $OUT
