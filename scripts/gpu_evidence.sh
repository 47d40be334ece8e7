#!/bin/bash
# Round evidence: GPU tests, the default bench line, the ncu launch list of the
# bench command, and one ncu --set full capture of the sweep and the Newton.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
for CFG in ${CFGS:-2 3}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 \
    -o gpurun_out/prof_sweep_${TAG}_c${CFG} -f python scripts/prof_step.py --config $CFG --warmup 3 --steps 1 > gpurun_out/prof_sweep_${TAG}_c${CFG}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_newton -s 3 -c 1 \
    -o gpurun_out/prof_newton_${TAG}_c${CFG} -f python scripts/prof_step.py --config $CFG --warmup 3 --steps 1 > gpurun_out/prof_newton_${TAG}_c${CFG}.log 2>&1
done
tail -3 gpurun_out/pytest_gpu_${TAG}.log; cat gpurun_out/bench_${TAG}.json
