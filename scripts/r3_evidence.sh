#!/bin/bash
# Round-2 evidence: smoke, GPU suite, default bench (config 4), its ncu launch
# list, bench lines of every workload, ncu --set full summaries of the hot kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-round2c}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=15 > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_bench_${TAG}.csv > gpurun_out/launches_bench_${TAG}.json
: > gpurun_out/bench_lines_${TAG}.jsonl
LINES=("--config 3" "--config 5" "--config 2 --steps 200" "--config 6 --steps 400" "--config 10 --steps 400"
       "--config 1 --steps 400" "--config 7 --steps 40" "--config 8 --steps 10" "--config 9 --steps 40"
       "--config 2 --tau sc --steps 100" "--config 2 --semi 100 --steps 100" "--config 2 --decomp band --steps 100"
       "--config 3 --implicit 4 --steps 2" "--config 2 --implicit 4 --steps 20" "--config 11 --steps 10")
for A in "${LINES[@]}"; do
  timeout 900 python bench.py $A --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> gpurun_out/bench_lines_${TAG}.jsonl
done
declare -A DOF=( [2]=230400000 [3]=4194304000 [4]=2000000000 [6]=15840000 [7]=460800000 [8]=3145728000 )
declare -A WL=( [2]=config2_2d_si_120x120x400x40 [3]="config3_3d_si_64^3x400x40" [4]="config4_3d_si_100^3x400x40" [6]=demo_2d_si_120x120x20x55 [7]=u2_tri_28800x400x40 [8]=u3_tet_196608x400x40 )
for CK in 4:sweep 4:newton 3:sweep 2:sweep 6:sweep 6:newton 7:usweep 8:usweep; do
  CFG=${CK%%:*}; K=${CK##*:}
  R=gpurun_out/prof_${K}_${TAG}_c${CFG}
  SKIP=3; [ $CFG = 4 ] && [ $K = sweep ] && SKIP=9
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_${K} -s $SKIP -c 1 \
    -o $R -f python scripts/prof_step.py --config $CFG --warmup 3 --steps 1 > $R.log 2>&1
  D=${DOF[$CFG]}
  python scripts/ncu_summary.py rep $R.ncu-rep --workload "${WL[$CFG]}" --dof $D > $R.json
  rm -f $R.ncu-rep
done
du -sh gpurun_out; tail -3 gpurun_out/pytest_gpu_${TAG}.log; cat gpurun_out/smoke_${TAG}.log; cut -c1-300 gpurun_out/bench_${TAG}.json
