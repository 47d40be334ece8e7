#!/bin/bash
# End-of-session evidence: smoke, GPU suite, default bench line (config 4), its launch list,
# bench lines of every workload.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-round2e}
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 2400 python -m pytest tests -m gpu -q -rfs --durations=10 > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_bench_${TAG}.csv > gpurun_out/launches_bench_${TAG}.json
rm -f gpurun_out/launches_bench_${TAG}.csv
: > gpurun_out/bench_lines_${TAG}.jsonl
LINES=("--config 3" "--config 5" "--config 2 --steps 200" "--config 6 --steps 400" "--config 10 --steps 400"
       "--config 1 --steps 400" "--config 7 --steps 40" "--config 8 --steps 10" "--config 9 --steps 40"
       "--config 2 --tau sc --steps 100" "--config 2 --semi 100 --steps 100" "--config 2 --decomp band --steps 100"
       "--config 3 --implicit 4 --steps 2" "--config 2 --implicit 4 --steps 20" "--config 11 --steps 10")
for A in "${LINES[@]}"; do
  timeout 900 python bench.py $A --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> gpurun_out/bench_lines_${TAG}.jsonl
done
tail -3 gpurun_out/pytest_gpu_${TAG}.log; cat gpurun_out/smoke_${TAG}.log; cut -c1-300 gpurun_out/bench_${TAG}.json
