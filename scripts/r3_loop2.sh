#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -rf > gpurun_out/pytest_loop2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_loop2.log
tail -5 gpurun_out/pytest_loop2.log
timeout 2400 python -m pytest tests -m gpu -q -rfs > gpurun_out/pytest_gpu_loop2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_loop2.log
tail -4 gpurun_out/pytest_gpu_loop2.log
