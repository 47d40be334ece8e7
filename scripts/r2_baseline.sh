#!/bin/bash
# Round 2 first call: current code's GPU suite, bench lines of configs 3/4, and
# the two-ranks-on-one-GPU NCCL probe.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2a}
timeout 600 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  scripts/nccl_same_gpu.py > gpurun_out/nccl_probe_${TAG}.log 2>&1; echo "exit $?" >> gpurun_out/nccl_probe_${TAG}.log
NCCL_DEBUG=WARN timeout 600 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  scripts/nccl_same_gpu.py > gpurun_out/nccl_probe2_${TAG}.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${TAG}.log
for A in "--config 3 --steps 20" "--config 4 --steps 6"; do
  N=$(echo $A | tr -d ' -')
  timeout 600 python bench.py $A --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_$N.json 2> gpurun_out/bench_${TAG}_$N.err
done
tail -3 gpurun_out/pytest_gpu_${TAG}.log; cat gpurun_out/nccl_probe_${TAG}.log | tail -8; cat gpurun_out/bench_${TAG}_*.json | cut -c1-400
