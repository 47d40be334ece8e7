#!/bin/bash
# Round 2 evidence call: smoke, the GPU suite, the default bench line (config 4,
# the north_star case), the ncu launch list of the bench command, and ncu
# --set full captures of the sweep on configs 4 and 3.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2b}
SKIP_TESTS=${SKIP_TESTS:-0}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
if [ "$SKIP_TESTS" = 0 ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
fi
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_bench_${TAG}.csv > gpurun_out/launches_bench_${TAG}.json
declare -A DOF=( [3]=4194304000 [4]=2000000000 )
declare -A WL=( [3]="config3_3d_si_64^3x400x40" [4]="config4_3d_si_100^3x400x40" )
for CFG in ${PROF_CFGS:-4 3}; do
  R=gpurun_out/prof_sweep_${TAG}_c${CFG}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 \
    -o $R -f python scripts/prof_step.py --config $CFG --warmup 3 --steps 1 > $R.log 2>&1
  python scripts/ncu_summary.py rep $R.ncu-rep --workload "${WL[$CFG]}" --dof ${DOF[$CFG]} > $R.json
  ncu -i $R.ncu-rep --page source --csv > $R.source.csv 2>/dev/null
  rm -f $R.ncu-rep
done
du -sh gpurun_out; tail -5 gpurun_out/pytest_gpu_${TAG}.log; cat gpurun_out/smoke_${TAG}.log; cut -c1-600 gpurun_out/bench_${TAG}.json
