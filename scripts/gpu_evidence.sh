#!/bin/bash
# Round evidence: GPU tests, the default bench line, the ncu launch list of the
# bench command, and one ncu --set full capture of the sweep and the Newton per
# config (summarised on the box with scripts/ncu_summary.py; only the config-2
# sweep report is kept to stay under gpurun's 64 MiB copy-back limit).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_bench_${TAG}.csv > gpurun_out/launches_bench_${TAG}.json
declare -A DOF=( [2]=230400000 [3]=4194304000 [6]=15840000 )
declare -A WL=( [2]=config2_2d_si_120x120x400x40 [3]="config3_3d_si_64^3x400x40" [6]=demo_2d_si_120x120x20x55 )
for CFG in ${CFGS:-2 3}; do
  for K in sweep newton; do
    R=gpurun_out/prof_${K}_${TAG}_c${CFG}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_${K} -s 3 -c 1 \
      -o $R -f python scripts/prof_step.py --config $CFG --warmup 3 --steps 1 > $R.log 2>&1
    python scripts/ncu_summary.py rep $R.ncu-rep --workload "${WL[$CFG]}" --dof ${DOF[$CFG]} > $R.json
    if [ "$K$CFG" != "sweep2" ]; then rm -f $R.ncu-rep; fi
  done
done
du -sh gpurun_out; tail -3 gpurun_out/pytest_gpu_${TAG}.log; cat gpurun_out/bench_${TAG}.json
