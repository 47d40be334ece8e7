#!/bin/bash
# Final evidence of the round: smoke, all GPU tests, the default bench line, the
# ncu launch list of the bench command, bench lines of the other workloads,
# ncu --set full summaries of the sweep and Newton (configs 2, 3) and of the
# unstructured sweep (u2, u3).  Reports are summarised on the box and deleted
# (gpurun copies back at most 64 MiB).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r05}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_bench_${TAG}.csv > gpurun_out/launches_bench_${TAG}.json
LINES=("--config 3 --steps 30" "--config 4 --steps 6" "--config 6 --steps 200" "--config 7 --steps 40"
       "--config 8 --steps 10" "--config 9 --steps 40" "--config 2 --tau sc --steps 100" "--config 2 --semi 100 --steps 200")
for A in "${LINES[@]}"; do
  N=$(echo $A | tr -d ' -')
  timeout 600 python bench.py $A --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$N.json 2> gpurun_out/bench_${TAG}_$N.err
done
declare -A DOF=( [2]=230400000 [3]=4194304000 [7]=460800000 [8]=3145728000 )
declare -A WL=( [2]=config2_2d_si_120x120x400x40 [3]="config3_3d_si_64^3x400x40" [7]=u2_tri_28800x400x40 [8]=u3_tet_196608x400x40 )
for CFG in 2 3 7 8; do
  for K in sweep newton; do
    [ $CFG -ge 7 ] && [ $K = newton ] && continue
    KR=$K; [ $CFG -ge 7 ] && KR=usweep
    R=gpurun_out/prof_${KR}_${TAG}_c${CFG}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_${KR} -s 3 -c 1 \
      -o $R -f python scripts/prof_step.py --config $CFG --warmup 3 --steps 1 > $R.log 2>&1
    python scripts/ncu_summary.py rep $R.ncu-rep --workload "${WL[$CFG]}" --dof ${DOF[$CFG]} > $R.json
    rm -f $R.ncu-rep
  done
done
du -sh gpurun_out; tail -3 gpurun_out/pytest_gpu_${TAG}.log; cat gpurun_out/bench_${TAG}.json
