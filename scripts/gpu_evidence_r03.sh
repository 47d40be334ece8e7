#!/bin/bash
# Round evidence (r03): smoke, all GPU tests, the default bench line, the ncu
# launch list of the bench command, bench lines of the other workloads, and
# ncu --set full summaries of the unstructured sweep and the self-consistent Newton.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r03}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_bench_${TAG}.csv > gpurun_out/launches_bench_${TAG}.json
for A in "--config 3 --steps 30" "--config 4 --steps 6" "--config 6 --steps 200" "--config 7 --steps 40" "--config 8 --steps 10" "--config 2 --tau sc --steps 100" "--config 2 --semi 100 --steps 200"; do
  N=$(echo $A | tr -d ' -')
  timeout 600 python bench.py $A --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}_$N.json 2> gpurun_out/bench_${TAG}_$N.err
done
for CFG in 7 8; do
  R=gpurun_out/prof_usweep_${TAG}_c${CFG}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_usweep -s 2 -c 1 \
    -o $R -f python scripts/prof_step.py --config $CFG --warmup 2 --steps 1 > $R.log 2>&1
  python scripts/ncu_summary.py rep $R.ncu-rep --workload c$CFG > $R.json
  rm -f $R.ncu-rep
done
R=gpurun_out/prof_newton_sc_${TAG}_c2
BTE_TAU_MODE=1 timeout 900 ncu --set full --clock-control none -k regex:k_newton -s 2 -c 1 \
  -o $R -f python scripts/prof_step.py --config 2 --warmup 2 --steps 1 --tau 1 > $R.log 2>&1
python scripts/ncu_summary.py rep $R.ncu-rep --workload config2 > $R.json
rm -f $R.ncu-rep
du -sh gpurun_out; tail -3 gpurun_out/pytest_gpu_${TAG}.log; cat gpurun_out/bench_${TAG}.json
