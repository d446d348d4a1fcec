#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_xchg.py -q -x > gpurun_out/pytest_xchg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_xchg.log
tail -30 gpurun_out/pytest_xchg.log
