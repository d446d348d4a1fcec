#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k gemv > gpurun_out/pytest_gemv.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gemv.log
tail -15 gpurun_out/pytest_gemv.log
timeout 300 python scripts/ab.py build/liblift_tma.so > gpurun_out/ab6.log 2>&1
cat gpurun_out/ab6.log
