#!/bin/bash
# compute-sanitizer passes (memcheck, racecheck, synccheck) over small GPU cases
# of every sweep family (structured TMA / plain, unstructured pipelined /
# plain, semi-implicit relax, sampled gather).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
OUT=gpurun_out/sanitize.txt
: > $OUT
CASES="${CASES:-tests/test_gpu_umesh.py::test_umesh_parity_all_wall_kinds tests/test_gpu_umesh.py::test_uquad_parity tests/test_gpu_parity.py::test_parity_small_3d_all_bc_kinds tests/test_gpu_parity.py::test_semi_parity tests/test_gpu_parity.py::test_parity_config1_full}"
for TOOL in ${TOOLS:-memcheck racecheck synccheck}; do
  for C in $CASES; do
    timeout 900 compute-sanitizer --tool $TOOL --error-exitcode 99 --print-limit 20 python -m pytest -q -x "$C" > gpurun_out/san_${TOOL}.log 2>&1
    rc=$?
    echo "$TOOL $C rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${TOOL}.log | tail -1)" >> $OUT
    [ $rc -ne 0 ] && cp gpurun_out/san_${TOOL}.log gpurun_out/san_${TOOL}_fail_$(echo $C | tr ':/' '__').log
  done
done
cat $OUT
