#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "asum or dot or fused or fuzz" > gpurun_out/pytest_red.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_red.log
timeout 600 python scripts/ab.py build/liblift_pfoff.so build/liblift_pfon.so build/liblift_pfoff.so build/liblift_pfon.so > gpurun_out/ab37.log 2>&1; cat gpurun_out/ab37.log
python scripts/trace_reduce.py 16777216 | head -12
