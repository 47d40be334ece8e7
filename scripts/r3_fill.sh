#!/bin/bash
# Streaming k_fill_eq: T-only set_state tests, full GPU suite, the default bench line (e2e), launch list.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-fill}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -rf -k "temperature_only" 2>&1 | tail -3
timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --repeats 1 --no-cpu-baseline > gpurun_out/launches_bench_${TAG}.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_bench_${TAG}.csv > gpurun_out/launches_bench_${TAG}.json
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e'], d['clocks'])"
